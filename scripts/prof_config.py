"""Per-class device time of one solve of a config (builders as configs_sweep)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import configs_sweep as CS  # noqa: E402
import paper_1703_07206_b200 as S  # noqa: E402
from paper_1703_07206_b200 import _capi  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
g, b, f, s, a = CS.fields(name, n)
ctx = S.Context(0)
grid = S.make_grid(g.dim, g.n)
bc = S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[i]), b.value[i]) for i in range(6)])
fd = S.Field.from_numpy(grid, f, ctx=ctx)
sd = S.Field.from_numpy(grid, s, ctx=ctx) if s is not None else None
ud = S.Field(grid, ctx=ctx)
slv = S.Solver(grid, bc, a=a, sigma=sd, config=S.SolverConfig(n_r=2, tol=1e-10, max_cycles=60, safety=0.9),
               options=S.SolverOptions(timing=True), ctx=ctx)
slv.run(fd, ud)
rep = slv.run(fd, ud)
rb = slv._rb.c
print(name, n, "cycles", len(rep.rows), "device_ms %.2f" % rep.device_ms, "launches", rep.kernel_launches)
for k, cname in enumerate(_capi.CLASS_NAMES[:7]):
    print("  %-13s %9.2f ms  %6d launches" % (cname, rb.class_ms[k], rb.class_launches[k]))
