"""Profiling driver: one solve of the capacitor (sigma) problem at 2^n+1 (device builders)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_07206_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 9
g = S.make_grid(3, n)
sig = S.capacitor_sigma(g, "high")
f = S.Field(g)
u = S.Field(g)
bc = S.BoundarySpec.all_neumann()
bc.set_face(2, 0, S.BcKind.dirichlet, -1.0)
bc.set_face(2, 1, S.BcKind.dirichlet, 1.0)
slv = S.Solver(g, bc, sigma=sig, config=S.SolverConfig(tol=1e-10, max_cycles=60),
               options=S.SolverOptions(timing=True))
rep = slv.run(f, u)
print("cycles", len(rep.rows), "final", rep.rows[-1].residual, "device_ms", rep.device_ms)
rb = slv._rb.c
for k, cname in enumerate(S._capi.CLASS_NAMES[:7]):
    print("  %-13s %9.2f ms  %6d launches" % (cname, rb.class_ms[k], rb.class_launches[k]))
