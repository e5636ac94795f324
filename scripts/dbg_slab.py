"""Debug: first trace entry where an in-process clique differs from the single-GPU solve."""
import sys
import threading
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import cases as K
import paper_1703_07206_b200 as S
from test_gpu_slabs import sgrid, sbc_of

name, n, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g, b, f, s, a = K.solve_problem(name, n)
prob = lambda: S.ProblemSpec(sgrid(g), f, bc=sbc_of(b), sigma=s, a=a)
cfg = S.SolverConfig(n_r=2, tol=1e-10, max_cycles=3, safety=0.9)
one = S.solve(prob(), cfg, ctx=S.Context(0))
grp = S.LocalGroup(P)
out = [None] * P
def run(r):
    c = S.Context(0); c.join_local(grp, r); out[r] = S.solve(prob(), cfg, ctx=c)
ts = [threading.Thread(target=run, args=(r,)) for r in range(P)]
[t.start() for t in ts]; [t.join() for t in ts]
t1 = [(t.cycle, t.pass_, t.level, t.value) for t in one.report.trace]
tp = [(t.cycle, t.pass_, t.level, t.value) for t in out[0].report.trace]
for i, (x, y) in enumerate(zip(t1, tp)):
    if x != y:
        print("first diff", i, x, y); break
else:
    print("traces equal", len(t1))
print("vrep", S.slab_plan(n, P, 0))
