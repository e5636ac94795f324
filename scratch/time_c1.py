import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_1703_07206_b200 as S
def run(dim, n, reps=20):
    g = S.make_grid(dim, n)
    f = S.sinsin2d_source(g) if dim == 2 else S.poisson3d_source(g)
    u = S.Field(g)
    slv = S.Solver(g, S.BoundarySpec.all_dirichlet(0.0), config=S.SolverConfig(tol=1e-10, max_cycles=60))
    for _ in range(3): rep = slv.run(f, u)
    ms = []
    for _ in range(reps):
        rep = slv.run(f, u); ms.append(rep.device_ms)
    return len(rep.rows), float(np.median(ms)), rep.kernel_launches
for dim, n in ((2, 7), (2, 8), (3, 6), (3, 7), (3, 9)):
    print(dim, n, run(dim, n, 20 if n < 9 else 5), flush=True)
