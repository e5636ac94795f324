"""Pin the C restatement (oracle/) before trusting it as the parity checker.

1. Known-answer residual histories measured from the reference
   (printed with %.17g).
2. Golden vectors produced by the UNMODIFIED reference
   (tests/golden/make_golden.py).
3. The live reference build (oracle/_ref) when this host has it.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import cases as K
from cases import O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
ARRAYS = np.load(os.path.join(HERE, "golden", "arrays.npz"))


def digest(a):
    return hashlib.sha256(K.canon(np.asarray(a, np.float64)).tobytes()).hexdigest()


# SURVEY.md 6.2, C1 literal sin-sin 129^2 and reference-native poisson2d_problem(7)
C1_SINSIN = [0.10873312228839256, 0.012156278408741049, 0.0012891593340796862,
             0.00013753723889625114, 1.4650998313436865e-05, 1.5611704034250908e-06,
             1.6634263726489735e-07, 1.7724058785398055e-08, 1.8885192779705005e-09,
             2.0122408249394345e-10, 2.1440673620972935e-11]
C1_POLY = [0.051960514853384328, 0.0044211470817878944, 0.00044864493935256556,
           4.7825538549201718e-05, 5.0841036478914009e-06, 5.4168657976540105e-07,
           5.7712901844465802e-08, 6.1493625740449153e-09, 6.5521998206200809e-10,
           6.981449114645922e-11]


@pytest.mark.parametrize("name,expect", [("sinsin2d", C1_SINSIN), ("poisson2d", C1_POLY)])
def test_known_answer_residual_histories(name, expect):
    g = O.make_grid(2, 7)
    res = O.solve(g, K.bc("dir0"), O.fill(name, g), tol=1e-10, max_cycles=60)
    assert res.converged
    assert [r[2] for r in res.rows] == expect  # bit-exact (%.17g round-trips)
    assert [r[1] for r in res.rows] == [114 * (i + 1) for i in range(len(expect))]


def test_golden_relax():
    for case in K.relax_cases(full=False):
        dim, n, level, bcn, sig, a, hom = case
        g, b, up, dup, gs, s = K.relax_inputs(*case)
        st, u, du, diag = O.relax(g, b, up, dup, level, gs, s, a, 0.9, hom)
        want = GOLDEN["relax"]["/".join(map(str, (dim, n, level, bcn, int(sig), a, int(hom))))]
        assert st == want["status"], case
        assert diag.hex() == want["diag"], case
        assert digest(u) == want["u"], case
        assert digest(du) == want["du"], case


def test_golden_arrays_roundtrip():
    # the full arrays agree with the digests (guards the fixture itself)
    for k in ARRAYS.files:
        kind, rest = k.split("/", 1)
        if kind == "relax_u":
            assert digest(ARRAYS[k]) == GOLDEN["relax"][rest]["u"]
        elif kind == "restriction":
            assert digest(ARRAYS[k]) == GOLDEN["restriction"][rest]["out"]


def test_golden_restriction():
    for dim, n in ((2, 4), (3, 3)):
        g = O.make_grid(dim, n)
        f = O.lcg(g, 11 + dim)
        for bcn in ("dir0", "neumann", "dir_distinct", "low_dir_high_neu"):
            for v in range(0, n + 1):
                r, w = O.restriction(g, K.bc(bcn), f, v)
                want = GOLDEN["restriction"][f"{dim}/{n}/{bcn}/{v}"]
                assert w == want["work"]
                assert digest(r) == want["out"], (dim, n, bcn, v)


def test_golden_residual():
    for dim, n in ((2, 4), (3, 3)):
        g = O.make_grid(dim, n)
        e = O.lcg(g, 23)
        f = O.lcg(g, 29)
        for bcn in ("dir0", "neumann", "dir_distinct", "low_dir_high_neu"):
            for sig in (False, True):
                for a in (0.0, 0.3):
                    s = K.sigma_field(g, 31) if sig else None
                    r = O.residual_update(g, K.bc(bcn), f, e, s, a)
                    assert digest(r) == GOLDEN["residual"][f"{dim}/{n}/{bcn}/{int(sig)}/{a}"]["r"]


@pytest.mark.parametrize("name,n", K.SOLVE_CASES)
def test_golden_solve(name, n):
    g, b, f, s, a = K.solve_problem(name, n)
    res = O.solve(g, b, f, s, a, n_r=2, tol=1e-10, max_cycles=40)
    want = GOLDEN["solve"][f"{name}/{n}"]
    assert [[c, w, r.hex(), d.hex()] for c, w, r, d in res.rows] == want["rows"]
    assert len(res.trace) == want["trace_len"]
    assert digest([t[3] for t in res.trace]) == want["trace"]
    assert digest(res.u) == want["u"]
    assert [res.converged, res.nan_detected, res.stagnated] == want["flags"]
    assert res.normalization.hex() == want["normalization"]
    assert res.node_updates == want["node_updates"]


def test_golden_schedule_units():
    for k, units in GOLDEN["schedule"].items():
        n, n_r = map(int, k.split("/"))
        assert O.closed_form_work_units(n, n_r) == units


needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="reference tree not on this host")


@needs_ref
def test_live_reference_relax_full_case_list():
    for case in K.relax_cases(full=True):
        dim, n, level, bcn, sig, a, hom = case
        g, b, up, dup, gs, s = K.relax_inputs(*case)
        mine = O.relax(g, b, up, dup, level, gs, s, a, 0.9, hom)
        ref = O.relax(g, b, up, dup, level, gs, s, a, 0.9, hom, impl="ref")
        # the reference's zero-weight corner reads past the end
        # of du_prev see zeros (oracle/ref_shim.cpp pads its allocations), the
        # value the restatement uses: every case must agree exactly
        assert mine[0] == ref[0] and mine[3] == ref[3], case
        assert K.bits_equal(mine[1], ref[1]) and K.bits_equal(mine[2], ref[2]), case


@needs_ref
@pytest.mark.parametrize("n_r", [1, 2, 3, 8])
def test_live_reference_single_cycle(n_r):
    for dim, n, bcn in ((2, 5, "mixed_x"), (3, 3, "plates"), (2, 4, "neumann")):
        g = O.make_grid(dim, n)
        src = O.lcg(g, 41 + n_r)
        sig = O.sigma_levels(g, K.sigma_field(g, 43))
        for levels in (None, sig):
            a = O.single_cycle(g, K.bc(bcn), src, levels, 0.2, False, n_r, 0.9, 0, 1.0)
            b = O.single_cycle(g, K.bc(bcn), src, levels, 0.2, False, n_r, 0.9, 0, 1.0, impl="ref")
            assert a[0] == b[0] and a[3] == b[3]
            assert K.bits_equal(a[1], b[1])
            assert [t[3] for t in a[2]] == [t[3] for t in b[2]]
            assert [t[:3] for t in a[2]] == [t[:3] for t in b[2]]


@needs_ref
def test_live_reference_problem_builders():
    g = O.make_grid(3, 4)
    _, _, f, _, _ = O.ref_problem("poisson3d", 4)
    assert K.bits_equal(f, O.fill("poisson3d", g))
    _, _, _, s, _ = O.ref_problem("capacitor_low", 4)
    assert K.bits_equal(s, O.fill("capacitor_sigma", g, 1.0))


@needs_ref
def test_live_reference_stagnation_and_validation():
    # indefinite a = 100 (cycle_tests.cpp:179-189) reports instead of throwing
    g = O.make_grid(2, 3)
    f = O.fill("poisson2d", g)
    a = O.solve(g, K.bc("dir0"), f, a=100.0, max_cycles=30)
    b = O.solve(g, K.bc("dir0"), f, a=100.0, max_cycles=30, impl="ref")
    assert (a.converged, a.nan_detected, a.stagnated) == (b.converged, b.nan_detected, b.stagnated)
    assert a.rows == b.rows and K.bits_equal(a.u, b.u)
    assert not a.converged
    bad = f.copy()
    bad[5] = float("nan")
    assert O.solve(g, K.bc("dir0"), bad).status == 1
    assert O.solve(g, K.bc("dir0"), bad, impl="ref").status == 1
