"""Debug helper: one compact single_cycle under the given parameters."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import cases as K
from cases import O
import paper_1703_07206_b200 as S

dim, n, bcn, n_r, sig, engine = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), sys.argv[5] == "1", sys.argv[6]
g = O.make_grid(dim, n)
sg = S.make_grid(dim, n)
src = O.lcg(g, 41 + n_r)
sfull = K.sigma_field(g, 43) if sig else None
kinds, vals = K.BCS[bcn]
bc = S.BoundarySpec([S.FaceBc(S.BcKind(k), float(v)) for k, v in zip(kinds, vals)])
slv = S.restrict_sigma_levels(S.Field.from_numpy(sg, sfull), n) if sig else []
state = S.SolveState(sg)
rep = S.SolveReport()
S.single_cycle(state, S.Field.from_numpy(sg, src), slv, 0.2, bc, False, S.build_schedule(n, n_r), 0.9, 3, 2.5, rep, S.Work(), S.SolverOptions(engine=engine))
st, u_ref, tr, w = O.single_cycle(g, K.bc(bcn), src, O.sigma_levels(g, sfull) if sig else None, 0.2, False, n_r, 0.9, 3, 2.5)
print("ok", K.bits_equal(state.u.numpy(), u_ref))
