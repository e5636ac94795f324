"""Compact 5/7-point stencil family.

The reference implements only the radial 9/27-point form; the north star
also names 5/7-point stencils.  This family is defined in the reference's
structure (axis offsets only, in the r, q, p order; inv_l2 = 1; prefactor 1;
Gershgorin step K = 1/(2d); the same sigma face average and ghosts).  PARITY
UNPINNED: there is no reference to compare with, so the C restatement is
validated by the properties SURVEY.md names (quadratic exactness, the
Gershgorin step, convergence), and the device is held bit-exact to the
restatement (GPU tests below).
"""
import numpy as np
import pytest

import cases as K
from cases import O
import paper_1703_07206_b200 as S


def coords(g):
    T = np.arange(g.total)
    return (T % g.N) * g.h, ((T // g.N) % g.N) * g.h, (T // (g.N * g.N)) * g.h


def apply_op(g, u, sigma=None):
    """A(u) of the compact form at interior nodes, through the residual update."""
    r = np.zeros(g.total)
    with O.stencil("compact"):
        O.c_lib().og_residual_update(O.C.byref(g), O.C.byref(O.all_neumann()), O._ptr(r), O._ptr(u),
                                     O._ptr(sigma), 0.0)
    return -r


@pytest.mark.parametrize("dim", [2, 3])
def test_compact_operator_exact_on_quadratics(dim):
    g = O.make_grid(dim, 4)
    x, y, z = coords(g)
    u = x * x + 2.0 * y * y + (3.0 * z * z if dim == 3 else 0.0)
    lap = 2.0 + 4.0 + (6.0 if dim == 3 else 0.0)
    a = apply_op(g, u).reshape((g.N,) * dim)
    assert np.all(a[(slice(1, -1),) * dim] == lap)
    # sigma constant 2: the operator scales by exactly 2
    a2 = apply_op(g, u, np.full(g.total, 2.0)).reshape((g.N,) * dim)
    assert np.all(a2[(slice(1, -1),) * dim] == 2.0 * lap)


@pytest.mark.parametrize("dim", [2, 3])
def test_compact_step_is_the_gershgorin_bound(dim):
    # one pass on a zero state with g = 0 except one node: the update is
    # u = dtau (0 - g) with dtau = safety K / (inv_s2 smax), K = 1/(2d)
    g = O.make_grid(dim, 3)
    gs = np.zeros(g.total)
    c = g.total // 2
    gs[c] = 1.0
    with O.stencil("compact"):
        st, u, du, diag = O.relax(g, O.all_dirichlet(0.0), np.zeros(g.total), np.zeros(g.total), 0, gs,
                                  None, 0.0, 0.9, False)
    K = 0.25 if dim == 2 else 1.0 / 6.0
    assert st == 0 and diag == 1.0
    assert u[c] == -(0.9 * K) / (1.0 / (g.h * g.h))


@pytest.mark.parametrize("name,n", [("sinsin2d", 6), ("poisson3d", 5), ("capacitor_low", 4), ("neumann2d_a", 5),
                                    ("mixed3d_a", 4)])
def test_compact_solves_converge(name, n):
    g, b, f, s, a = K.solve_problem(name, n)
    with O.stencil("compact"):
        res = O.solve(g, b, f, s, a, tol=1e-10, max_cycles=80)
    assert res.converged and not res.nan_detected
    assert res.rows[-1][2] <= 1e-10


def test_compact_discretisation_error_is_second_order():
    # manufactured sin-sin: the l_inf error against the exact solution drops ~4x per refinement
    errs = []
    for n in (4, 5, 6):
        g = O.make_grid(2, n)
        x, y, _ = coords(g)
        exact = np.sin(np.pi * x) * np.sin(np.pi * y)
        f = -2.0 * np.pi ** 2 * exact
        with O.stencil("compact"):
            res = O.solve(g, O.all_dirichlet(0.0), f, tol=1e-12, max_cycles=80)
        errs.append(np.max(np.abs(res.u - exact)))
    assert 3.5 < errs[0] / errs[1] < 4.5 and 3.5 < errs[1] / errs[2] < 4.5


def test_radial_stays_the_default():
    g, b, f, s, a = K.solve_problem("sinsin2d", 5)
    r1 = O.solve(g, b, f, tol=1e-10)
    with O.stencil("radial"):
        r2 = O.solve(g, b, f, tol=1e-10)
    assert r1.rows == r2.rows


# ------------------------------------------------------------------ GPU ----

def sbc_of(b):
    return S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[f]), b.value[f]) for f in range(6)])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["compact", "literal"])
@pytest.mark.parametrize("name,n", [("sinsin2d", 5), ("poisson2d", 6), ("poisson3d", 4), ("capacitor_high", 3),
                                    ("capacitor_low", 4), ("neumann2d_a", 4), ("mixed2d", 5), ("mixed3d_a", 3),
                                    ("sigma3d_dirichlet", 3), ("zero_source_dirichlet1", 3), ("neumann3d_a", 3)])
def test_compact_solve_bitwise_on_device(name, n, engine):
    g, b, f, s, a = K.solve_problem(name, n)
    with O.stencil("compact"):
        ref = O.solve(g, b, f, s, a, tol=1e-10, max_cycles=80)
    res = S.solve(S.ProblemSpec(S.make_grid(g.dim, g.n), f, bc=sbc_of(b), sigma=s, a=a),
                  S.SolverConfig(tol=1e-10, max_cycles=80), S.SolverOptions(engine=engine, stencil="compact"))
    rep = res.report
    assert (rep.converged, rep.nan_detected, rep.stagnated) == (ref.converged, ref.nan_detected, ref.stagnated)
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in rep.rows] == ref.rows
    assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == ref.trace
    assert K.bits_equal(res.u, ref.u)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n,bcn", [(2, 5, "mixed_x"), (3, 3, "plates"), (3, 4, "dir_distinct")])
@pytest.mark.parametrize("sig", [False, True])
def test_compact_single_cycle_bitwise_on_device(dim, n, bcn, sig):
    g = O.make_grid(dim, n)
    src = O.lcg(g, 71)
    sfull = K.sigma_field(g, 73) if sig else None
    levels = O.sigma_levels(g, sfull) if sig else None
    for hom in (False, True):
        with O.stencil("compact"):
            st, u_ref, trace_ref, w_ref = O.single_cycle(g, K.bc(bcn), src, levels, 0.2, hom, 2, 0.9, 1, 2.0)
        assert st == 0
        state = S.SolveState(S.make_grid(dim, n))
        rep = S.SolveReport()
        work = S.Work(0)
        slv = S.restrict_sigma_levels(S.Field.from_numpy(S.make_grid(dim, n), sfull), n) if sig else []
        S.single_cycle(state, S.Field.from_numpy(S.make_grid(dim, n), src), slv, 0.2,
                       S.BoundarySpec([S.FaceBc(S.BcKind(k), float(v)) for k, v in zip(*K.BCS[bcn])]), hom,
                       S.build_schedule(n, 2), 0.9, 1, 2.0, rep, work, S.SolverOptions(stencil="compact"))
        assert work.value == w_ref
        assert K.bits_equal(state.u.numpy(), u_ref)
        assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == trace_ref
