"""GPU parity on every relaxation-kernel specialisation the solve launches,
and on solves large enough that the TMA kernels (not the one-CTA small-level
path) carry sigma, a != 0, all-Neumann and mixed faces.

* k_relax_tma<DIM, SIG, HAS_A, MODE, DUO, CMP>: the matrix below runs every
  combination (dim x sigma x a x stencil family; relax passes with and
  without du output, the residual recurrence with u_tot) with the small-level
  path switched off (SolverOptions.small_levels = False), so every level
  runs through the TMA kernel, against the C restatement bit for bit.
* SOLVE_CASES_LARGE and SPEC_CASES (every specialisation at 2D 129^2 /
  3D 33^3, including x-high Dirichlet faces next to Neumann rows): the
  device against golden results produced by the
  UNMODIFIED reference (tests/golden/solves.json, make_golden_large.py
  --solves): residual history (hex), flags, normalisation, node updates,
  trace digest, solution digest.  Small-level path on and off.
* n_r = 128 (2D 257^2): a visit adding more pending increments than the
  materialisation keeps in shared memory (kMaxChain), and the fold of a
  long chain into a full-grid base.
"""
import functools
import hashlib
import json
import os

import numpy as np
import pytest

import cases as K
from cases import O
import paper_1703_07206_b200 as S

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SOLVES_JSON = os.path.join(HERE, "golden", "solves.json")


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert S.device_count() >= 1, "no CUDA device: GPU tests must run on the B200 box"
    S.default_context()


def sbc_of(b):
    return S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[f]), b.value[f]) for f in range(6)])


def digest(a) -> str:
    return hashlib.sha256(K.canon(np.asarray(a, np.float64)).tobytes()).hexdigest()


BCS = {2: ["dir_distinct", "neumann", "mixed_x"], 3: ["dir_distinct", "neumann", "low_dir_high_neu", "xdir_yzneu"]}


@pytest.mark.parametrize("stencil", ["radial", "compact"])
@pytest.mark.parametrize("a", [0.0, 0.25])
@pytest.mark.parametrize("sig", [False, True])
@pytest.mark.parametrize("dim,bci", [(d, i) for d in (2, 3) for i in range(len(BCS[d]))])
def test_every_tma_specialisation_bitwise(dim, bci, sig, a, stencil):
    n = 5 if dim == 2 else 4
    g = O.make_grid(dim, n)
    b = K.bc(BCS[dim][bci])
    f = O.fill("sinsin2d" if dim == 2 else "poisson3d", g)
    s = K.sigma_field(g, 57 + dim) if sig else None
    with O.stencil(stencil):
        ref = O.solve(g, b, f, s, a, n_r=2, tol=1e-10, max_cycles=25)
    res = S.solve(S.ProblemSpec(S.make_grid(dim, n), f, bc=sbc_of(b), sigma=s, a=a),
                  S.SolverConfig(n_r=2, tol=1e-10, max_cycles=25, safety=0.9),
                  S.SolverOptions(stencil=stencil, small_levels=False))
    rep = res.report
    assert (rep.converged, rep.nan_detected, rep.stagnated) == (ref.converged, ref.nan_detected, ref.stagnated)
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in rep.rows] == ref.rows
    assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == ref.trace
    assert K.bits_equal(res.u, ref.u)


@functools.lru_cache(maxsize=1)
def golden_solves():
    if not os.path.exists(SOLVES_JSON):
        return {}
    return json.load(open(SOLVES_JSON))


def check_against_golden(key, g, b, f, s, a, small_levels):
    gold = golden_solves().get(key)
    assert gold is not None, f"tests/golden/solves.json lacks {key} (make_golden_large.py --solves)"
    n = g.n
    assert digest(f) == gold["f"]
    res = S.solve(S.ProblemSpec(S.make_grid(g.dim, n), f, bc=sbc_of(b), sigma=s, a=a),
                  S.SolverConfig(n_r=2, tol=1e-10, max_cycles=60, safety=0.9),
                  S.SolverOptions(small_levels=small_levels))
    rep = res.report
    assert [rep.converged, rep.nan_detected, rep.stagnated] == gold["flags"]
    assert [[r.cycle, r.work_units, r.residual.hex(), r.diag_min.hex()] for r in rep.rows] == gold["rows"]
    assert rep.normalization.hex() == gold["normalization"]
    assert rep.node_updates == gold["node_updates"]
    assert len(rep.trace) == gold["trace_len"]
    assert digest([t.value for t in rep.trace]) == gold["trace"]
    assert digest(res.u) == gold["u"]


@pytest.mark.parametrize("small_levels", [True, False])
@pytest.mark.parametrize("name,n", K.SOLVE_CASES_LARGE, ids=lambda x: str(x))
def test_large_solves_match_reference_golden(name, n, small_levels):
    g, b, f, s, a = K.solve_problem(name, n)
    check_against_golden(f"case:{name}@{n}", g, b, f, s, a, small_levels)


@pytest.mark.parametrize("small_levels", [True, False])
@pytest.mark.parametrize("case", K.SPEC_CASES, ids=lambda c: K.spec_key(*c))
def test_specialisations_at_size_match_reference_golden(case, small_levels):
    g, b, f, s, a = K.spec_problem(*case)
    check_against_golden(K.spec_key(*case) + f"@{case[1]}", g, b, f, s, a, small_levels)


@pytest.mark.parametrize("engine,small_levels", [("compact", True), ("compact", False), ("literal", True)])
def test_single_cycle_long_chains_bitwise(engine, small_levels):
    # 2D 257^2, n_r = 128: tooth v1 = 2 relaxes 64 passes per level (the
    # pending chain outgrows kMaxChain = 96 and is folded into a full-grid
    # base); tooth v1 = 1 adds 127 increments in one visit, all applied by the
    # level-0 materialisation (entries past kMaxChain read from global memory)
    n, n_r = 8, 128
    g = O.make_grid(2, n)
    src = O.lcg(g, 71)
    for hom in (False, True):
        st, u_ref, trace_ref, w_ref = O.single_cycle(g, K.bc("mixed_x"), src, None, 0.1, hom, n_r, 0.9, 0, 1.5)
        assert st == 0
        state = S.SolveState(S.make_grid(2, n))
        rep = S.SolveReport()
        work = S.Work()
        S.single_cycle(state, S.Field.from_numpy(S.make_grid(2, n), src), [], 0.1, sbc_of(K.bc("mixed_x")), hom,
                       S.build_schedule(n, n_r), 0.9, 0, 1.5, rep, work,
                       S.SolverOptions(engine=engine, small_levels=small_levels))
        assert work.value == w_ref
        assert [t.value for t in rep.trace] == [t[3] for t in trace_ref]
        assert K.bits_equal(state.u.numpy(), u_ref)


def test_solve_long_chains_bitwise():
    g, b, f, s, a = K.solve_problem("sinsin2d", 7)
    ref = O.solve(g, b, f, s, a, n_r=100, tol=1e-10, max_cycles=6)
    res = S.solve(S.ProblemSpec(S.make_grid(2, 7), f, bc=sbc_of(b)),
                  S.SolverConfig(n_r=100, tol=1e-10, max_cycles=6, safety=0.9))
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in res.report.rows] == ref.rows
    assert K.bits_equal(res.u, ref.u)


# Tiny lattices (N = 3, 5, 9): one interior node, levels that exist only as
# faces, a single level, every boundary mix, sigma and a, on each engine path
# (compact with and without the interpreter and small-level visits, literal).
TINY_ENGINES = {
    "compact": dict(),
    "compact-nointerp": dict(cluster_levels=False),
    "compact-nosmall-nointerp": dict(cluster_levels=False, small_levels=False),
    "literal": dict(engine="literal"),
}


@pytest.mark.parametrize("engine", list(TINY_ENGINES))
@pytest.mark.parametrize("a", [0.0, 0.3])
@pytest.mark.parametrize("sig", [False, True])
@pytest.mark.parametrize("dim,n,bcn", [(d, n, b) for d, ns in ((2, (1, 2, 3)), (3, (1, 2, 3)))
                                       for n in ns for b in BCS[d]])
def test_tiny_lattices_bitwise(dim, n, bcn, sig, a, engine):
    g = O.make_grid(dim, n)
    b = K.bc(bcn)
    f = O.fill("sinsin2d" if dim == 2 else "poisson3d", g)
    s = K.sigma_field(g, 57 + dim) if sig else None
    ref = O.solve(g, b, f, s, a, n_r=2, tol=1e-10, max_cycles=25)
    res = S.solve(S.ProblemSpec(S.make_grid(dim, n), f, bc=sbc_of(b), sigma=s, a=a),
                  S.SolverConfig(n_r=2, tol=1e-10, max_cycles=25, safety=0.9),
                  S.SolverOptions(**TINY_ENGINES[engine]))
    rep = res.report
    assert (rep.converged, rep.nan_detected, rep.stagnated) == (ref.converged, ref.nan_detected, ref.stagnated)
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in rep.rows] == ref.rows
    assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == ref.trace
    assert K.bits_equal(res.u, ref.u)


# Other relaxation counts and safety factors where the TMA kernels carry the
# large levels (2D 129^2, 3D 33^3); tol 1e-12 with max_cycles 6 also exits
# on the cycle cap.
@pytest.mark.parametrize("n_r,safety,tol,max_cycles", [(1, 0.9, 1e-10, 40), (3, 0.9, 1e-10, 40),
                                                        (4, 0.6, 1e-10, 40), (2, 1.0, 1e-12, 6)])
@pytest.mark.parametrize("sig", [False, True])
@pytest.mark.parametrize("dim,n,bcn", [(2, 7, "mixed_x"), (3, 5, "dir_distinct"), (3, 5, "neumann")])
def test_relax_counts_and_safety_bitwise(dim, n, bcn, sig, n_r, safety, tol, max_cycles):
    g = O.make_grid(dim, n)
    b = K.bc(bcn)
    f = O.fill("sinsin2d" if dim == 2 else "poisson3d", g)
    s = K.sigma_field(g, 57 + dim) if sig else None
    a = 0.25 if bcn == "neumann" else 0.0
    ref = O.solve(g, b, f, s, a, n_r=n_r, tol=tol, max_cycles=max_cycles, safety=safety)
    res = S.solve(S.ProblemSpec(S.make_grid(dim, n), f, bc=sbc_of(b), sigma=s, a=a),
                  S.SolverConfig(n_r=n_r, tol=tol, max_cycles=max_cycles, safety=safety))
    rep = res.report
    assert (rep.converged, rep.nan_detected, rep.stagnated) == (ref.converged, ref.nan_detected, ref.stagnated)
    assert [(r.cycle, r.work_units, r.residual, r.diag_min) for r in rep.rows] == ref.rows
    assert [(t.cycle, t.pass_, t.level, t.value) for t in rep.trace] == ref.trace
    assert K.bits_equal(res.u, ref.u)
