"""Profiling driver: `runs` solves of a 3D problem at 2^n+1 (default 257^3).

    python scripts/prof_solve.py n runs [engine] [poisson|capacitor]

poisson: poisson3d_problem(n) (the bench problem); capacitor:
capacitor_problem(n, "high") (sigma, lateral Neumann).  Inputs are built on
the device; the first solve also captures the cycle graphs.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_07206_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
engine = sys.argv[3] if len(sys.argv) > 3 else "compact"
problem = sys.argv[4] if len(sys.argv) > 4 else "poisson"
timing = os.environ.get("SGML_PROF_TIMING", "0") == "1"
grid = S.make_grid(3, n)
u = S.Field(grid)
opts = S.SolverOptions(engine=engine, timing=timing)
cfg = S.SolverConfig(tol=1e-10, max_cycles=60)
if problem == "poisson":
    f = S.poisson3d_source(grid)
    slv = S.Solver(grid, S.BoundarySpec.all_dirichlet(0.0), config=cfg, options=opts)
else:
    f = S.Field(grid)
    bc = S.BoundarySpec.all_neumann()
    bc.set_face(2, 0, S.BcKind.dirichlet, -1.0)
    bc.set_face(2, 1, S.BcKind.dirichlet, 1.0)
    slv = S.Solver(grid, bc, sigma=S.capacitor_sigma(grid, "high"), config=cfg, options=opts)
for _ in range(runs):
    rep = slv.run(f, u)
print("cycles", len(rep.rows), "final", rep.rows[-1].residual, "device_ms", rep.device_ms)
if timing:
    from paper_1703_07206_b200 import _capi
    c = slv._rb.c
    for k, name in enumerate(_capi.CLASS_NAMES[:7]):
        print(f"  {name:14s} {c.class_ms[k]:9.3f} ms  {int(c.class_launches[k]):6d} launches")
