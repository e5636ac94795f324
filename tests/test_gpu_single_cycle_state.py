"""single_cycle with the reference's full SolveState semantics:
the C++ drop-in's single_cycle (sgml_single_cycle_state) against the
UNMODIFIED reference (oracle/_ref) on states that do not start at zero,
schedules other than build_schedule's, sigma levels that are not a
restriction pyramid, and a pass that overflows mid-cycle.  Everything the
reference leaves behind is compared bit for bit: u, u_prev, du, du_prev,
level, the trace and the work counter."""
import numpy as np
import pytest

import cases as K
from cases import O
import paper_1703_07206_b200 as S

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(O.ref_lib() is None, reason="reference build (oracle/_ref) unavailable")]


def sbc_of(b):
    return S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[f]), b.value[f]) for f in range(6)])


SCHEDULES = {
    "built": None,  # build_schedule(n, 2)
    # relax at level 1 before any restriction (g still zero), repeated and
    # out-of-order levels, a restriction to level 0, a level revisited
    "custom": [(1, 1, 2), (0, 2, 1), (1, 2, 3), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1), (1, 1, 2)],
}


def run_both(dim, n, bcn, sched_name, with_sigma, hom, scale=1.0, safety=0.9):
    g = O.make_grid(dim, n)
    b = K.bc(bcn)
    src = scale * O.lcg(g, 301)
    u0, up0, du0, dup0 = (O.lcg(g, s) for s in (303, 305, 307, 309))
    levels = None
    if with_sigma:  # arbitrary positive levels, not a restriction pyramid
        levels = np.stack([1.0 + 0.5 * np.abs(O.lcg(g, 311 + v)) for v in range(g.n)])
    steps = SCHEDULES[sched_name] or [(st[0], st[1], st[2]) for st in O.build_schedule(n, 2)]
    ref = O.ref_single_cycle_state(g, b, u0, up0, du0, dup0, 3, src, levels, 0.2, hom, steps, safety, 4, 2.5, 11)

    sg = S.make_grid(dim, n)
    state = S.SolveState(sg)
    for f, arr in zip((state.u, state.u_prev, state.du, state.du_prev), (u0, up0, du0, dup0)):
        f.upload(arr)
    state.level = 3
    lv = [S.Field.from_numpy(sg, levels[v]) for v in range(g.n)] if with_sigma else []
    sched = S.CycleSchedule(n, 2, [S.ScheduleStep(k, l, c) for k, l, c in steps])
    rep, work = S.SolveReport(), S.Work(11)
    err = None
    try:
        S.single_cycle_state(state, S.Field.from_numpy(sg, src), lv, 0.2, sbc_of(b), hom, sched, safety, 4, 2.5,
                             rep, work)
    except S.kernel_error as e:
        err = e
    return ref, (err, state, rep, work)


@pytest.mark.parametrize("hom", [False, True])
@pytest.mark.parametrize("with_sigma", [False, True])
@pytest.mark.parametrize("sched", ["built", "custom"])
@pytest.mark.parametrize("dim,n,bcn", [(2, 4, "mixed_x"), (3, 3, "plates"), (2, 3, "dir_distinct")])
def test_single_cycle_state_matches_reference(dim, n, bcn, sched, with_sigma, hom):
    (st, u, up, du, dup, level, trace, work_ref), (err, state, rep, work) = run_both(dim, n, bcn, sched,
                                                                                      with_sigma, hom)
    assert st == 0 and err is None
    assert K.bits_equal(state.u.numpy(), u) and K.bits_equal(state.u_prev.numpy(), up)
    assert K.bits_equal(state.du.numpy(), du) and K.bits_equal(state.du_prev.numpy(), dup)
    assert state.level == level
    assert work.value == work_ref
    assert [(t.cycle, t.pass_, t.level) for t in rep.trace] == [t[:3] for t in trace]
    assert [t.value for t in rep.trace] == [t[3] for t in trace]


@pytest.mark.parametrize("dim,n,bcn", [(2, 5, "dir0"), (3, 3, "dir_distinct")])
def test_single_cycle_state_failing_pass_leaves_the_reference_state(dim, n, bcn):
    (st, u, up, du, dup, level, trace, work_ref), (err, state, rep, work) = run_both(
        dim, n, bcn, "built", False, False, scale=1e300, safety=20.0)
    assert st != 0 and err is not None
    assert K.bits_equal(state.u.numpy(), u) and K.bits_equal(state.u_prev.numpy(), up)
    assert K.bits_equal(state.du.numpy(), du) and K.bits_equal(state.du_prev.numpy(), dup)
    assert state.level == level and work.value == work_ref
    assert [t.value for t in rep.trace] == [t[3] for t in trace]
