"""Profiling driver: one warm-up solve + one solve of 3D Poisson at 2^n+1 (default 257^3)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (for the source builder)
import paper_1703_07206_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
engine = sys.argv[3] if len(sys.argv) > 3 else "compact"
grid = S.make_grid(3, n)
f = S.Field.from_numpy(grid, bench.poisson3d_source(n))
u = S.Field(grid)
slv = S.Solver(grid, S.BoundarySpec.all_dirichlet(0.0), config=S.SolverConfig(tol=1e-10),
               options=S.SolverOptions(engine=engine, timing=True))
for _ in range(runs):
    rep = slv.run(f, u)
print("cycles", len(rep.rows), "final", rep.rows[-1].residual, "device_ms", rep.device_ms)
