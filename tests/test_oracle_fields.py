"""Pin the C restatement of the post-solve operators (oracle/sgml_oracle.c,
problems.cpp:40-97, 327-455) before it checks the device kernels.

1. Golden digests produced by the UNMODIFIED reference
   (tests/golden/make_golden.py, section "fields").
2. The reference's own unit / acceptance expectations for these functions
   (problems_tests.cpp:165-309, acceptance_main.cpp:270-309).
3. The live reference build (oracle/_ref) when this host has it.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import cases as K
from cases import O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))["fields"]


def digest(a):
    return hashlib.sha256(K.canon(np.asarray(a, np.float64)).tobytes()).hexdigest()


def coords(g):
    T = np.arange(g.total)
    return (T % g.N) * g.h, ((T // g.N) % g.N) * g.h, (T // (g.N * g.N)) * g.h


@pytest.mark.parametrize("dim,n", K.FIELD_GRIDS)
def test_golden_fields(dim, n):
    d = K.field_inputs(dim, n)
    g = d["g"]
    want = GOLDEN[f"{dim}/{n}"]
    assert digest(O.gradient(g, d["u"])) == want["gradient"]
    assert digest(O.divergence(g, d["v"])) == want["divergence"]
    if dim == 3:
        assert digest(O.curl(g, d["psi"])) == want["curl"]
    st, vel = O.deformation_velocity(g, d["u"], d["f_raw"], d["raw_integral"], d["t"])
    assert [st, digest(vel)] == want["deformation_velocity"]
    st, pos = O.move_nodes(g, 0.01 * d["u"], d["f_raw"], d["raw_integral"], d["t"], d["steps"])
    assert [st, digest(pos)] == want["move_nodes"]
    lines = []
    for field in ("swirl", "v"):
        for seed in d["seeds"]:
            pts, stop = O.integrate_streamline(g, d[field], seed, d["step"], d["max_steps"])
            lines.append([field, len(pts), stop, digest(pts)])
    assert lines == want["streamlines"]
    assert [digest(O.sample_vector(g, d["v"], p)) for p in d["seeds"]] == want["sample"]


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 3), (3, 5)])
def test_live_reference_fields(dim, n):
    if O.ref_lib() is None:
        pytest.skip("reference build unavailable on this host")
    rng = np.random.default_rng(7 + n)
    g = O.make_grid(dim, n)
    u = rng.standard_normal(g.total)
    v = rng.standard_normal((dim, g.total))
    f_raw = np.abs(rng.standard_normal(g.total))
    assert K.bits_equal(O.gradient(g, u), O.gradient(g, u, impl="ref"))
    assert K.bits_equal(O.divergence(g, v), O.divergence(g, v, impl="ref"))
    if dim == 3:
        psi = rng.standard_normal((3, g.total))
        assert K.bits_equal(O.curl(g, psi), O.curl(g, psi, impl="ref"))
    a = O.deformation_velocity(g, u, f_raw, 0.7, 0.2)
    b = O.deformation_velocity(g, u, f_raw, 0.7, 0.2, impl="ref")
    assert a[0] == b[0] and K.bits_equal(a[1], b[1])
    a = O.move_nodes(g, 0.02 * u, f_raw, 0.7, 0.4, 9)
    b = O.move_nodes(g, 0.02 * u, f_raw, 0.7, 0.4, 9, impl="ref")
    assert a[0] == b[0] and K.bits_equal(a[1], b[1])
    seed = [0.41, 0.57, 0.5 if dim == 3 else 0.0]
    p1, s1 = O.integrate_streamline(g, v, seed, 0.01, 200)
    p2, s2 = O.integrate_streamline(g, v, seed, 0.01, 200, impl="ref")
    assert s1 == s2 and K.bits_equal(p1, p2)


# ---- the reference's own expectations (problems_tests.cpp) ----------------

def test_deformation_velocity_divides_the_gradient():
    # problems_tests.cpp:165-175
    g = O.make_grid(2, 3)
    x, _, _ = coords(g)
    u = 2.0 * x
    f_raw = np.zeros(g.total)
    st, v = O.deformation_velocity(g, u, f_raw, 4.0, 0.7)
    p = 3 + g.N * 3
    assert st == 0 and v[0][p] == pytest.approx(-0.5, rel=1e-13) and abs(v[1][p]) <= 1e-13
    assert O.deformation_velocity(g, u, f_raw, 0.0, 0.0)[0] == 1


def test_move_nodes_flat_potential():
    # problems_tests.cpp:177-189
    g = O.make_grid(2, 2)
    st, pos = O.move_nodes(g, np.zeros(g.total), np.zeros(g.total), 1.0, 0.5, 10)
    x, y, _ = coords(g)
    assert st == 0
    assert np.allclose(pos[:, 0], x, rtol=1e-15) and np.allclose(pos[:, 1], y, rtol=1e-15)
    assert O.move_nodes(g, np.zeros(g.total), np.zeros(g.total), 1.0, 0.5, 0)[0] == 1


def test_difference_fields_exact_on_quadratics():
    # problems_tests.cpp:214-252
    g = O.make_grid(3, 3)
    x, y, z = coords(g)
    grad = O.gradient(g, x * x + 2.0 * y)
    assert np.allclose(grad[0], 2.0 * x, atol=1e-12) and np.allclose(grad[1], 2.0, atol=1e-12)
    assert np.allclose(grad[2], 0.0, atol=1e-12)
    v = O.curl(g, np.stack([y * y, z * z, x * x]))
    assert np.allclose(v[0], -2.0 * z, atol=1e-12)
    assert np.allclose(v[1], -2.0 * x, atol=1e-12)
    assert np.allclose(v[2], -2.0 * y, atol=1e-12)


def test_divergence_of_curl_vanishes():
    # problems_tests.cpp:253-265
    g = O.make_grid(3, 4)
    x, y, z = coords(g)
    psi = np.stack([np.sin(math.pi * y) * np.cos(2 * math.pi * z), np.exp(x) * np.sin(math.pi * z),
                    np.cos(math.pi * x) * y * y])
    assert np.max(np.abs(O.divergence(g, O.curl(g, psi)))) <= 1e-12


def test_streamline_stop_conditions():
    # problems_tests.cpp:281-309
    g = O.make_grid(2, 3)
    drift = np.stack([np.ones(g.total), np.zeros(g.total)])
    pts, stop = O.integrate_streamline(g, drift, [0.75, 0.5, 0.0], 0.1, 100)
    assert stop == 1 and len(pts) >= 2 and pts[1][0] == pytest.approx(0.85, rel=1e-13)
    pts, stop = O.integrate_streamline(g, np.zeros((2, g.total)), [0.5, 0.5, 0.0], 0.1, 100)
    assert stop == 2 and len(pts) == 1
    x, y, _ = coords(g)
    spin = np.stack([-(y - 0.5), x - 0.5])
    pts, stop = O.integrate_streamline(g, spin, [0.7, 0.5, 0.0], 0.01, 500)
    assert stop == 0 and len(pts) == 501


def test_rk4_orbit_closes():
    # acceptance_main.cpp:287-309 (criterion 8, second half)
    g = O.make_grid(2, 5)
    x, y, _ = coords(g)
    om = 2.0 * 3.14159265358979323846 / 6.0
    rot = np.stack([-om * (y - 0.5), om * (x - 0.5)])
    pts, stop = O.integrate_streamline(g, rot, [0.75, 0.5, 0.0], 1e-3, 6000)
    assert stop == 0 and len(pts) == 6001
    assert math.hypot(pts[-1][0] - 0.75, pts[-1][1] - 0.5) <= 1e-6


def test_sample_vector_multilinear_exact():
    # problems_tests.cpp:266-279
    g = O.make_grid(2, 3)
    x, y, _ = coords(g)
    v = np.stack([3.0 * x - y, 0.5 + y])
    s = O.sample_vector(g, v, [0.317, 0.682, 0.0])
    assert s[0] == pytest.approx(3.0 * 0.317 - 0.682, rel=1e-12)
    assert s[1] == pytest.approx(0.5 + 0.682, rel=1e-12) and s[2] == 0.0
