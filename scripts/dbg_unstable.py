"""Debug: reports of solves that blow up (overflow mid-cycle) vs the oracle."""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import cases as K
from cases import O
import paper_1703_07206_b200 as S
for name, n, safety, scale in (("poisson3d", 4, 20.0, 1e300), ("sinsin2d", 5, 30.0, 1e305), ("poisson3d", 4, 0.9, 1e308),
                               ("capacitor_high", 3, 50.0, 1.0), ("sinsin2d", 5, 0.9, 1e308)):
    g, b, f, s, a = K.solve_problem(name, n)
    f = f * scale
    if name == "capacitor_high":
        b = O.make_bc(list(b.kind), [0, 0, 0, 0, -1e308, 1e308])
    if not np.isfinite(f).all():
        print(name, scale, "source overflows; skipped"); continue
    ref = O.solve(g, b, f, s, a, tol=1e-10, max_cycles=40, safety=safety)
    bc = S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[i]), b.value[i]) for i in range(6)])
    res = S.solve(S.ProblemSpec(S.make_grid(g.dim, g.n), f, bc=bc, sigma=s, a=a),
                  S.SolverConfig(tol=1e-10, max_cycles=40, safety=safety))
    r = res.report
    print(name, safety, scale, "trace eq", [(t.cycle, t.pass_, t.level, t.value) for t in r.trace] == ref.trace, "ref", ref.converged, ref.nan_detected, ref.stagnated, len(ref.rows), len(ref.trace),
          "| ours", r.converged, r.nan_detected, r.stagnated, len(r.rows), len(r.trace),
          "| rows eq", [(x.cycle, x.work_units, x.residual, x.diag_min) for x in r.rows] == ref.rows)
