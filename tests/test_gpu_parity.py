"""GPU parity: the sm_100a path (through the C-ABI) against the oracle.

Bar: bit-identical fp64 results, with -0.0 folded into +0.0 (SURVEY.md
8(c); the device skips zero-weight interpolation corners, which can only
flip the sign of an exact zero).  The oracle is oracle/'s C restatement,
itself pinned to the reference by tests/test_oracle_pinning.py.
"""
import math

import numpy as np
import pytest

import cases as K
from cases import O
import paper_1703_07206_b200 as S

pytestmark = pytest.mark.gpu


def sgrid(g):
    return S.make_grid(g.dim, g.n)


def sbc(name):
    kinds, vals = K.BCS[name]
    return S.BoundarySpec([S.FaceBc(S.BcKind(k), float(v)) for k, v in zip(kinds, vals)])


def dev(g, arr):
    return S.Field.from_numpy(sgrid(g), arr)


# engine variants: the compact engine with and without the one-CTA
# small-level path (SolverOptions.small_levels) and the small-level cluster
# interpreter (cluster_levels; "compact-kopall": interpreted up to 65^3-node
# levels, SGML_KOP_NODES), and the literal engine
ENGINES = ["compact", "compact-nosmall", "compact-nocluster", "compact-kopall", "literal"]


@pytest.fixture(autouse=True)
def _kop_env(request, monkeypatch):
    if "compact-kopall" in request.node.name:
        monkeypatch.setenv("SGML_KOP_NODES", str(65 ** 3))


def opts(engine):
    return S.SolverOptions(engine="literal" if engine == "literal" else "compact",
                           small_levels=engine != "compact-nosmall",
                           cluster_levels=engine not in ("compact-nosmall", "compact-nocluster"))


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert S.device_count() >= 1, "no CUDA device: GPU tests must run on the B200 box"
    S.default_context()


# ------------------------------------------------------------ kernels ----

@pytest.mark.parametrize("case", K.relax_cases(full=True), ids=lambda c: "-".join(map(str, c)))
def test_relaxation_interpolation_bitwise(case):
    dim, n, level, bcn, sig, a, hom = case
    g, b, up, dup, gs, s = K.relax_inputs(*case)
    st, u_ref, du_ref, diag_ref = O.relax(g, b, up, dup, level, gs, s, a, 0.9, hom)
    state = S.SolveState(sgrid(g))
    state.level = level
    state.u_prev.upload(up)
    state.du_prev.upload(dup)
    work = S.Work()
    diag = S.relaxation_interpolation(state, dev(g, gs), dev(g, s) if sig else None, a, 0.9,
                                      sbc(bcn), hom, work)
    assert st == 0
    assert work.value == 1
    assert diag == diag_ref
    assert K.bits_equal(state.u.numpy(), u_ref)
    assert K.bits_equal(state.du.numpy(), du_ref)


def test_relaxation_kernel_error_on_nan_and_badstep():
    # kernels_tests.cpp:160-169
    g = O.make_grid(2, 2)
    state = S.SolveState(sgrid(g))
    up = np.zeros(g.total)
    up[12] = np.nan
    state.u_prev.upload(up)
    with pytest.raises(S.kernel_error):
        S.relaxation_interpolation(state, dev(g, np.zeros(g.total)), None, 0.0, 0.9, sbc("dir0"), True)
    with pytest.raises(S.kernel_error):
        S.relaxation_interpolation(S.SolveState(sgrid(g)), dev(g, np.zeros(g.total)), None, 0.0, 0.0,
                                   sbc("dir0"), True)


@pytest.mark.parametrize("dim,n", [(2, 4), (2, 6), (3, 3), (3, 5)])
@pytest.mark.parametrize("bcn", ["dir0", "neumann", "dir_distinct", "low_dir_high_neu"])
def test_restriction_into_bitwise(dim, n, bcn):
    g = O.make_grid(dim, n)
    f = O.lcg(g, 11 + dim)
    fd = dev(g, f)
    for v in range(0, n + 1):
        ref, w_ref = O.restriction(g, K.bc(bcn), f, v)
        work = S.Work()
        out = S.restriction(fd, v, sbc(bcn), work)
        assert work.value == w_ref
        assert K.bits_equal(out.numpy(), ref), v


@pytest.mark.parametrize("dim,n", [(2, 4), (2, 7), (3, 3), (3, 5)])
@pytest.mark.parametrize("bcn", ["dir0", "neumann", "dir_distinct", "low_dir_high_neu"])
@pytest.mark.parametrize("sig", [False, True])
@pytest.mark.parametrize("a", [0.0, 0.3])
def test_residual_update_bitwise(dim, n, bcn, sig, a):
    g = O.make_grid(dim, n)
    e = O.lcg(g, 23)
    f = O.lcg(g, 29)
    s = K.sigma_field(g, 31) if sig else None
    ref = O.residual_update(g, K.bc(bcn), f, e, s, a)
    r = dev(g, f)
    S.residual_update(r, dev(g, e), S.OperatorCoefficients(dev(g, s) if sig else None, a), sbc(bcn))
    assert K.bits_equal(r.numpy(), ref)


def test_max_abs_trapezoid_projection():
    for dim, n in ((2, 5), (3, 4)):
        g = O.make_grid(dim, n)
        f = O.lcg(g, 31) + 2.0
        fd = dev(g, f)
        assert S.max_abs(fd) == O.c_lib().og_max_abs(O._ptr(f), g.total)
        assert S.trapezoid_mean(fd) == O.c_lib().og_trapezoid_mean(O.C.byref(g), O._ptr(f))
        S.zero_mean_projection(fd)
        ref = f.copy()
        O.c_lib().og_zero_mean_projection(O.C.byref(g), O._ptr(ref))
        assert K.bits_equal(fd.numpy(), ref)


def test_apply_boundary_matches_oracle():
    g = O.make_grid(3, 3)
    for hom in (False, True):
        u = O.lcg(g, 5)
        ref = u.copy()
        O.c_lib().og_apply_boundary(O.C.byref(g), O.C.byref(K.bc("dir_distinct")), O._ptr(ref), int(hom))
        ud = dev(g, u)
        S.apply_boundary(ud, sbc("dir_distinct"), hom)
        assert K.bits_equal(ud.numpy(), ref)


def test_restrict_sigma_levels_and_positivity():
    g = O.make_grid(2, 4)
    s = K.sigma_field(g, 3)
    levels = S.restrict_sigma_levels(dev(g, s), g.n)
    ref = O.sigma_levels(g, s).reshape(g.n, -1)
    for v in range(g.n):
        assert K.bits_equal(levels[v].numpy(), ref[v])
    bad = s.copy()
    bad[40] = -50.0
    with pytest.raises(ValueError):
        S.restrict_sigma_levels(dev(g, bad), g.n)


# -------------------------------------------------------------- cycle ----

@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("n_r", [1, 2, 3, 8])
@pytest.mark.parametrize("dim,n,bcn", [(2, 5, "mixed_x"), (3, 3, "plates"), (2, 4, "neumann"),
                                       (3, 4, "dir_distinct"), (2, 1, "dir0"), (3, 2, "low_dir_high_neu")])
@pytest.mark.parametrize("sig", [False, True])
def test_single_cycle_bitwise(engine, n_r, dim, n, bcn, sig):
    g = O.make_grid(dim, n)
    src = O.lcg(g, 41 + n_r)
    sfull = K.sigma_field(g, 43) if sig else None
    levels = O.sigma_levels(g, sfull) if sig else None
    for hom in (False, True):
        st, u_ref, trace_ref, w_ref = O.single_cycle(g, K.bc(bcn), src, levels, 0.2, hom, n_r, 0.9, 3,
                                                     2.5)
        assert st == 0
        state = S.SolveState(sgrid(g))
        rep = S.SolveReport()
        work = S.Work(7)
        slv = S.restrict_sigma_levels(dev(g, sfull), g.n) if sig else []
        S.single_cycle(state, dev(g, src), slv, 0.2, sbc(bcn), hom, S.build_schedule(n, n_r), 0.9, 3,
                       2.5, rep, work, opts(engine))
        assert work.value == 7 + w_ref
        assert K.bits_equal(state.u.numpy(), u_ref)
        assert [(t.cycle, t.pass_, t.level) for t in rep.trace] == [t[:3] for t in trace_ref]
        assert [t.value for t in rep.trace] == [t[3] for t in trace_ref]


# -------------------------------------------------------------- solve ----

def check_solve(name, n, engine="compact", n_r=2, tol=1e-10, max_cycles=40):
    g, b, f, s, a = K.solve_problem(name, n)
    ref = O.solve(g, b, f, s, a, n_r=n_r, tol=tol, max_cycles=max_cycles)
    prob = S.ProblemSpec(sgrid(g), f, bc=sbc_of(b), sigma=s, a=a)
    res = S.solve(prob, S.SolverConfig(n_r=n_r, tol=tol, max_cycles=max_cycles, safety=0.9), opts(engine))
    rep = res.report
    assert (rep.converged, rep.nan_detected, rep.stagnated) == (ref.converged, ref.nan_detected,
                                                                ref.stagnated)
    assert len(rep.rows) == len(ref.rows)
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in rep.rows] == ref.rows
    assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == ref.trace
    assert rep.normalization == ref.normalization
    assert rep.node_updates == ref.node_updates
    assert K.bits_equal(res.u, ref.u)
    return res, ref


def sbc_of(b):
    return S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[f]), b.value[f]) for f in range(6)])


@pytest.mark.parametrize("name,n", K.SOLVE_CASES, ids=lambda x: str(x))
@pytest.mark.parametrize("engine", ENGINES)
def test_solve_bitwise(name, n, engine):
    check_solve(name, n, engine)


@pytest.mark.parametrize("n_r", [1, 3, 8])
def test_solve_other_relax_counts(n_r):
    check_solve("sinsin2d", 5, n_r=n_r)
    check_solve("capacitor_low", 3, n_r=n_r)


def test_solve_c1_config_known_answer():
    # BASELINE.json configs[0]: 2D 129^2 sin-sin; SURVEY.md 6.2 history
    res, _ = check_solve("sinsin2d", 7)
    assert len(res.report.rows) == 11
    assert res.report.rows[0].residual == 0.10873312228839256
    assert res.report.rows[-1].residual == 2.1440673620972935e-11


@pytest.mark.parametrize("scale", [2.0 ** -1000, 2.0 ** -1062])
@pytest.mark.parametrize("name,n", [("poisson3d", 4), ("sinsin2d", 5)])
def test_solve_tiny_values_bitwise(name, n, scale):
    # values near the subnormal range: the relaxation kernels must drop the
    # fused edge terms (flag[1]) and still match the reference bit for bit
    g, b, f, s, a = K.solve_problem(name, n)
    f = f * scale
    ref = O.solve(g, b, f, s, a, tol=1e-10, max_cycles=12)
    res = S.solve(S.ProblemSpec(sgrid(g), f, bc=sbc_of(b), sigma=s, a=a),
                  S.SolverConfig(n_r=2, tol=1e-10, max_cycles=12, safety=0.9))
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in res.report.rows] == ref.rows
    # a subnormal normalisation turns some diagnostics into inf / nan (both sides)
    same = lambda x, y: x == y or (math.isnan(x) and math.isnan(y))  # noqa: E731
    got = [(t.cycle, t.pass_, t.level, t.value) for t in res.report.trace]
    assert len(got) == len(ref.trace)
    assert all(a[:3] == b[:3] and same(a[3], b[3]) for a, b in zip(got, ref.trace))
    assert K.bits_equal(res.u, ref.u)


def test_solve_tiny_dirichlet_value_bitwise():
    g = O.make_grid(3, 4)
    f = O.fill("poisson3d", g)
    b = O.make_bc([0, 0, 0, 0, 0, 0], [2.0 ** -1000, 0.0, 0.0, 0.0, 0.0, 3e-310])
    ref = O.solve(g, b, f, tol=1e-10, max_cycles=12)
    res = S.solve(S.ProblemSpec(sgrid(g), f, bc=sbc_of(b)),
                  S.SolverConfig(n_r=2, tol=1e-10, max_cycles=12, safety=0.9))
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in res.report.rows] == ref.rows
    assert K.bits_equal(res.u, ref.u)


@pytest.mark.parametrize("engine", ["compact", "literal"])
@pytest.mark.parametrize("name,n,safety,scale", [
    ("poisson3d", 4, 20.0, 1e300), ("sinsin2d", 5, 30.0, 1e305), ("capacitor_high", 3, 50.0, 1.0),
    ("poisson3d", 5, 40.0, 1e250), ("sinsin2d", 6, 10.0, 1e200), ("sinsin2d", 6, 3.0, 1e300),
    ("poisson3d", 5, 4.0, 1e300), ("neumann3d_a", 4, 20.0, 1e250),
    # failing in cycle 2 / 1 (after rows were recorded): the recurrence ran
    # before the host saw the failure and skipped itself (guarded residual)
    ("poisson3d", 4, 2.0, 1e300), ("sinsin2d", 5, 3.0, 1e290)])
def test_solve_overflow_partial_trace(name, n, safety, scale, engine):
    # a pass that overflows mid-cycle throws kernel_error in the reference
    # (kernels.cpp:343-346): nan_detected, no row for the cycle, and the trace
    # keeps the samples of the passes before the failing one (cycle.cpp:98-107)
    g, b, f, s, a = K.solve_problem(name, n)
    f = f * scale
    if name == "capacitor_high":
        b = O.make_bc(list(b.kind), [0, 0, 0, 0, -1e308, 1e308])
    ref = O.solve(g, b, f, s, a, tol=1e-10, max_cycles=40, safety=safety)
    res = S.solve(S.ProblemSpec(sgrid(g), f, bc=sbc_of(b), sigma=s, a=a),
                  S.SolverConfig(tol=1e-10, max_cycles=40, safety=safety), S.SolverOptions(engine=engine))
    rep = res.report
    assert (rep.converged, rep.nan_detected, rep.stagnated) == (ref.converged, ref.nan_detected, ref.stagnated)
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in rep.rows] == ref.rows
    assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == ref.trace
    assert K.bits_equal(res.u, ref.u)


@pytest.mark.parametrize("engine", ["compact", "literal"])
@pytest.mark.parametrize("name,n,safety,scale", [
    ("poisson3d", 4, 20.0, 1e300), ("sinsin2d", 6, 3.0, 1e300), ("capacitor_high", 3, 50.0, 1.0)])
def test_single_cycle_overflow_partial_trace(name, n, safety, scale, engine):
    # single_cycle throws at the failing pass with the samples and work units
    # of the steps before it already recorded (cycle.cpp:88-107)
    g, b, f, s, a = K.solve_problem(name, n)
    f = f * scale
    if name == "capacitor_high":
        b = O.make_bc(list(b.kind), [0, 0, 0, 0, -1e308, 1e308])
    levels = O.sigma_levels(g, s) if s is not None else None
    st, _, trace_ref, w_ref = O.single_cycle(g, b, f, levels, a, False, 2, safety, 0, 1.0)
    assert st != 0
    state = S.SolveState(sgrid(g))
    rep = S.SolveReport()
    work = S.Work(3)
    slv = S.restrict_sigma_levels(dev(g, s), g.n) if s is not None else []
    with pytest.raises(S.kernel_error):
        S.single_cycle(state, dev(g, f), slv, a, sbc_of(b), False, S.build_schedule(n, 2), safety, 0, 1.0,
                       rep, work, S.SolverOptions(engine=engine))
    assert work.value == 3 + w_ref
    assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == trace_ref


def test_solve_larger_3d():
    check_solve("poisson3d", 6)          # 65^3
    check_solve("capacitor_high", 5)     # 33^3, sigma + mixed faces


def test_solve_indefinite_reports_instead_of_throwing():
    # cycle_tests.cpp:179-189
    g = O.make_grid(2, 3)
    f = O.fill("poisson2d", g)
    ref = O.solve(g, K.bc("dir0"), f, a=100.0, max_cycles=30)
    res = S.solve(S.ProblemSpec(sgrid(g), f, bc=sbc("dir0"), a=100.0), S.SolverConfig(max_cycles=30))
    assert not res.report.converged
    assert (res.report.stagnated, res.report.nan_detected) == (ref.stagnated, ref.nan_detected)
    assert [r.residual for r in res.report.rows] == [r[2] for r in ref.rows]
    assert K.bits_equal(res.u, ref.u)


def test_solve_validates_inputs():
    # cycle_tests.cpp:191-202
    g = O.make_grid(2, 3)
    f = O.fill("poisson2d", g)
    prob = S.ProblemSpec(sgrid(g), f, bc=sbc("dir0"))
    with pytest.raises(ValueError):
        S.solve(prob, S.SolverConfig(tol=0.0))
    with pytest.raises(ValueError):
        S.solve(prob, S.SolverConfig(n_r=0))
    bad = f.copy()
    bad[10] = np.nan
    with pytest.raises(ValueError):
        S.solve(S.ProblemSpec(sgrid(g), bad, bc=sbc("dir0")), S.SolverConfig())
    sig = np.ones(g.total)
    sig[30] = -50.0
    with pytest.raises(ValueError):
        S.solve(S.ProblemSpec(sgrid(g), f, bc=sbc("dir0"), sigma=sig), S.SolverConfig())


def test_solve_tol_one_stops_after_one_cycle():
    g = O.make_grid(2, 4)
    res = S.solve(S.ProblemSpec(sgrid(g), O.fill("poisson2d", g), bc=sbc("dir0")),
                  S.SolverConfig(tol=1.0))
    assert res.report.converged and len(res.report.rows) == 1


def test_solver_object_repeated_runs_identical():
    g = O.make_grid(3, 5)
    f = O.fill("poisson3d", g)
    slv = S.Solver(sgrid(g), sbc("dir0"), config=S.SolverConfig(tol=1e-10))
    fd = dev(g, f)
    u1 = S.Field(sgrid(g))
    u2 = S.Field(sgrid(g))
    r1 = slv.run(fd, u1)
    r2 = slv.run(fd, u2)
    assert [r.residual for r in r1.rows] == [r.residual for r in r2.rows]
    assert K.bits_equal(u1.numpy(), u2.numpy())
    ref = O.solve(g, K.bc("dir0"), f, tol=1e-10)
    assert K.bits_equal(u1.numpy(), ref.u)


def test_solve_twice_with_nonzero_dirichlet_values():
    # the cached engine's buffers keep their face contents between solves
    # (u_tot picks up the face values in cycle 0 of every solve)
    for name, n in (("capacitor_high", 3), ("capacitor_low", 3), ("sigma3d_dirichlet", 3)):
        for _ in range(2):
            check_solve(name, n)


@pytest.mark.parametrize("name,n", [("poisson3d", 4), ("capacitor_high", 3), ("sinsin2d", 5)])
def test_solve_many_equals_single_solves(name, n):
    # sgml_solve_many pipelines the transfers of neighbouring solves; each
    # result must be the single solve's, bit for bit
    g, b, f, s, a = K.solve_problem(name, n)
    scales = [1.0, -0.5, 3.0] if not np.all(f == 0) else [1.0]
    probs = [S.ProblemSpec(sgrid(g), f * c, bc=sbc_of(b), sigma=s, a=a) for c in scales]
    cfg = S.SolverConfig(tol=1e-10, max_cycles=40)
    many = S.solve_many(probs, cfg)
    for p, m in zip(probs, many):
        one = S.solve(p, cfg)
        assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in m.report.rows] == \
            [(r.cycle, r.work_units, r.residual, r.diag_min) for r in one.report.rows]
        assert [(t.cycle, t.pass_, t.level, t.value) for t in m.report.trace] == \
            [(t.cycle, t.pass_, t.level, t.value) for t in one.report.trace]
        assert np.array_equal(m.u.view(np.int64), one.u.view(np.int64))
