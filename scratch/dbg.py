import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import cases as K
from cases import O
import paper_1703_07206_b200 as S

def sbc_of(b):
    return S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[f]), b.value[f]) for f in range(6)])

def run(g, b, f, s, a, n_r=2, small=True):
    n = g.n
    levels = O.sigma_levels(g, s) if s is not None else None
    st, u_ref, tr_ref, w_ref = O.single_cycle(g, b, f, levels, a, False, n_r, 0.9, 0, 1.0)
    state = S.SolveState(S.make_grid(g.dim, n)); rep = S.SolveReport(); work = S.Work()
    slv = S.restrict_sigma_levels(S.Field.from_numpy(S.make_grid(g.dim, n), s), g.n) if s is not None else []
    S.single_cycle(state, S.Field.from_numpy(S.make_grid(g.dim, n), f), slv, a, sbc_of(b), False,
                   S.build_schedule(n, n_r), 0.9, 0, 1.0, rep, work, S.SolverOptions(small_levels=small))
    u = state.u.numpy()
    tr = [t.value for t in rep.trace]
    bad = [i for i, (x, y) in enumerate(zip(tr, [t[3] for t in tr_ref])) if x != y]
    d = np.abs(u - u_ref).reshape((g.N,) * g.dim)
    idx = np.argwhere(d > 0)
    return K.bits_equal(u, u_ref), bad[:1], ([tr_ref[i][2] for i in bad[:1]]), idx[:6].tolist(), len(idx)

D, N = O.DIRICHLET, O.NEUMANN
for n in (7, 8):
    g = O.make_grid(2, n)
    for kinds in ([D,D,N,N],[N,N,D,D],[D,N,N,N],[N,D,N,N],[D,D,D,N],[D,D,N,D],[N,N,D,N],[N,N,N,D],[N,N,N,N]):
        b = O.make_bc(kinds + [N, N], [0.5, -0.75, 0.25, 0.125, 0, 0])
        for n_r in (1, 2):
            print(n, kinds, n_r, run(g, b, O.fill("sinsin2d", g), None, 0.0, n_r=n_r), flush=True)
