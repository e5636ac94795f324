import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_1703_07206_b200 as S
from paper_1703_07206_b200 import _capi
g = S.make_grid(2, 7)
f = S.sinsin2d_source(g); u = S.Field(g)
for opts in (S.SolverOptions(timing=True), S.SolverOptions(timing=True, use_graph=False)):
    slv = S.Solver(g, S.BoundarySpec.all_dirichlet(0.0), config=S.SolverConfig(tol=1e-10), options=opts)
    for _ in range(3): rep = slv.run(f, u)
    c = slv._rb.c
    print("device_ms", rep.device_ms, "launches", rep.kernel_launches, "graph", opts.use_graph)
    for k, name in enumerate(_capi.CLASS_NAMES[:7]):
        print(f"  {name:14s} {c.class_ms[k]:8.3f} ms {int(c.class_launches[k]):5d}")
slv = S.Solver(g, S.BoundarySpec.all_dirichlet(0.0), config=S.SolverConfig(tol=1e-10))
for _ in range(3): rep = slv.run(f, u)
print("untimed device_ms", rep.device_ms)
