import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_1703_07206_b200 as S
from oracle import oracle as O
import cases as K
for n in (2, 3):
    g = O.make_grid(2, n)
    src = O.fill("sinsin2d", g)
    res = {}
    for eng in ("compact", "literal"):
        state = S.SolveState(S.make_grid(2, n)); rep = S.SolveReport(); work = S.Work(0)
        f = S.Field.from_numpy(S.make_grid(2, n), src)
        S.single_cycle(state, f, [], 0.0, S.BoundarySpec.all_dirichlet(0.0), False, S.build_schedule(n, 1), 0.9, 0, 0.0, rep, work, S.SolverOptions(engine=eng))
        res[eng] = ([(t.pass_, t.level, t.value) for t in rep.trace], state.u.numpy())
    for a, b in zip(res["compact"][0], res["literal"][0]):
        print(n, a, b, "OK" if a == b else "DIFF")
    print(np.abs(res["compact"][1] - res["literal"][1]).max())
