"""GPU parity of the post-solve operators (csrc/fields.cu) against the
pinned C restatement (tests/test_oracle_fields.py): bit-identical fp64,
-0.0 folded into +0.0."""
import math

import numpy as np
import pytest

import cases as K
from cases import O
import paper_1703_07206_b200 as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert S.device_count() >= 1, "no CUDA device: GPU tests must run on the B200 box"
    S.default_context()


def sgrid(g):
    return S.make_grid(g.dim, g.n)


def dev(g, a):
    return S.Field.from_numpy(sgrid(g), a)


def vdev(g, arrays):
    return S.VectorField.from_numpy(sgrid(g), arrays)


GRIDS = K.FIELD_GRIDS + [(2, 7), (3, 6)]


@pytest.mark.parametrize("dim,n", GRIDS)
def test_difference_fields_bitwise(dim, n):
    d = K.field_inputs(dim, n)
    g = d["g"]
    u = dev(g, d["u"])
    for axis in range(dim):
        assert K.bits_equal(S.axis_derivative(u, axis).numpy(), O.axis_derivative(g, d["u"], axis))
    grad = S.gradient(u).numpy()
    assert K.bits_equal(grad[:dim], O.gradient(g, d["u"]))
    assert K.bits_equal(S.divergence(vdev(g, d["v"])).numpy(), O.divergence(g, d["v"]))
    if dim == 3:
        assert K.bits_equal(S.curl(vdev(g, d["psi"])).numpy(), O.curl(g, d["psi"]))
    else:
        with pytest.raises(ValueError):
            S.curl(vdev(g, d["psi"][:2]))


@pytest.mark.parametrize("dim,n", GRIDS)
def test_deformation_velocity_and_move_nodes_bitwise(dim, n):
    d = K.field_inputs(dim, n)
    g = d["g"]
    st, vel = O.deformation_velocity(g, d["u"], d["f_raw"], d["raw_integral"], d["t"])
    assert st == 0
    got = S.deformation_velocity(dev(g, d["u"]), dev(g, d["f_raw"]), d["raw_integral"], d["t"]).numpy()
    assert K.bits_equal(got[:dim], vel)
    u = 0.01 * d["u"]
    st, pos = O.move_nodes(g, u, d["f_raw"], d["raw_integral"], d["t"], d["steps"])
    got = S.move_nodes(dev(g, u), dev(g, d["f_raw"]), d["raw_integral"], d["t"], d["steps"]).numpy()
    assert K.bits_equal(got.T, pos)


def test_field_errors_follow_the_reference():
    g = O.make_grid(2, 3)
    x = (np.arange(g.total) % g.N) * g.h
    u, z = dev(g, 2.0 * x), dev(g, np.zeros(g.total))
    with pytest.raises(ValueError):  # problems.cpp:334-335
        S.deformation_velocity(u, z, 0.0, 0.0)
    with pytest.raises(ValueError):  # problems.cpp:345
        S.move_nodes(u, z, 1.0, 0.5, 0)
    with pytest.raises(ValueError):  # problems.cpp:417
        S.integrate_streamline(S.gradient(u), [0.5, 0.5, 0.0], 0.0, 10)


@pytest.mark.parametrize("dim,n", GRIDS)
def test_streamlines_and_samples_bitwise(dim, n):
    d = K.field_inputs(dim, n)
    g = d["g"]
    for name in ("swirl", "v"):
        v = vdev(g, d[name])
        lines = S.integrate_streamlines(v, d["seeds"], d["step"], d["max_steps"])
        for seed, line in zip(d["seeds"], lines):
            pts, stop = O.integrate_streamline(g, d[name], seed, d["step"], d["max_steps"])
            assert int(line.stop) == stop
            assert K.bits_equal(line.points, pts)
        got = S.sample_vector(v, d["seeds"])
        want = np.stack([O.sample_vector(g, d[name], p) for p in d["seeds"]])
        assert K.bits_equal(got, want)


def test_rk4_orbit_closes_on_device():
    # acceptance_main.cpp:287-309
    g = O.make_grid(2, 5)
    T = np.arange(g.total)
    x, y = (T % g.N) * g.h, ((T // g.N) % g.N) * g.h
    om = 2.0 * 3.14159265358979323846 / 6.0
    rot = np.stack([-om * (y - 0.5), om * (x - 0.5)])
    line = S.integrate_streamline(vdev(g, rot), [0.75, 0.5, 0.0], 1e-3, 6000)
    pts, stop = O.integrate_streamline(g, rot, [0.75, 0.5, 0.0], 1e-3, 6000)
    assert line.stop == S.StreamlineStop.max_steps and len(line.points) == 6001
    assert K.bits_equal(line.points, pts)
    assert math.hypot(line.points[-1][0] - 0.75, line.points[-1][1] - 0.5) <= 1e-6


def test_div_curl_of_solved_potentials():
    # acceptance_main.cpp:270-286 at a small size: psi from three device
    # solves of the knotted-vortex problem, div(curl psi) ~ 0 inside
    if O.ref_lib() is None:
        pytest.skip("trifoil sources come from the reference build (oracle/_ref)")
    comps = []
    for c in "xyz":
        g, b, f, s, a = O.ref_problem("trifoil_" + c, 4)
        res = S.solve(S.ProblemSpec(sgrid(g), f, bc=S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[i]), b.value[i])
                                                                    for i in range(6)])),
                      S.SolverConfig(tol=1e-10, max_cycles=60))
        assert res.report.converged
        comps.append(res.u)
    psi = vdev(g, comps)
    div = S.divergence(S.curl(psi)).numpy().reshape(g.N, g.N, g.N)
    assert np.max(np.abs(div[1:-1, 1:-1, 1:-1])) <= 1e-13
    assert K.bits_equal(S.curl(psi).numpy(), O.curl(g, np.stack(comps)))


# ---- problem builders on the device ------------------

@pytest.mark.parametrize("n", [3, 5, 8])
def test_device_builders_match_the_reference_bits(n):
    g3 = O.make_grid(3, n)
    assert K.bits_equal(S.poisson3d_source(sgrid(g3)).numpy(), O.fill("poisson3d", g3))
    for mode, sign in (("high", -1.0), ("low", 1.0)):
        assert K.bits_equal(S.capacitor_sigma(sgrid(g3), mode).numpy(), O.fill("capacitor_sigma", g3, sign))
    g2 = O.make_grid(2, n + 2)
    assert K.bits_equal(S.poisson2d_source(sgrid(g2)).numpy(), O.fill("poisson2d", g2))
    assert K.bits_equal(S.sinsin2d_source(sgrid(g2)).numpy(), O.fill("sinsin2d", g2))


@pytest.mark.parametrize("n", [3, 5, 7])
def test_device_curve_sources_match_the_reference(n):
    if O.ref_lib() is None:
        pytest.skip("curve sources are compared with the reference build (oracle/_ref)")
    g = O.make_grid(3, n)
    fs = S.trifoil_sources(sgrid(g), 0.14)
    for c, name in enumerate("xyz"):
        _, _, f, _, _ = O.ref_problem("trifoil_" + name, n)
        got = fs[c].numpy()
        assert np.array_equal(got.view(np.int64), f.view(np.int64))  # incl. the -0.0 of the negation
    t = 2.0 * 3.14159265358979323846 * np.arange(32) / 32.0
    pts = np.stack([0.5 + 0.25 * np.cos(t), 0.5 + 0.25 * np.sin(t), np.zeros(32)], axis=1)
    g2 = O.make_grid(2, n + 3)
    f, f_raw, ri = S.deformation_sources(pts, sgrid(g2))
    gr, f_raw_ref, f_ref, ri_ref = O.ref_deformation_setup(pts, 0.1, n + 3)
    assert ri == ri_ref
    assert K.bits_equal(f_raw.numpy(), f_raw_ref) and K.bits_equal(f.numpy(), f_ref)


# ---- streamed VTK output (io.cpp:14-64) ---------------

@pytest.mark.parametrize("dim,n", [(2, 4), (3, 3), (3, 5)])
def test_streamed_vtk_matches_the_reference_bytes(dim, n, tmp_path):
    if O.ref_lib() is None:
        pytest.skip("the byte reference is the reference's own writer (oracle/_ref)")
    g = O.make_grid(dim, n)
    rng = np.random.default_rng(n)
    u = rng.standard_normal(g.total) * 10.0 ** rng.integers(-300, 300, g.total)
    u[:5] = [0.0, -0.0, 1.0, 0.1, 1e-320]
    S.write_field_vtk(dev(g, u), tmp_path / "a.vtk", "u")
    O.ref_lib().ref_write_field_vtk(O.C.byref(g), O._ptr(u), str(tmp_path / "b.vtk").encode(), b"u")
    assert (tmp_path / "a.vtk").read_bytes() == (tmp_path / "b.vtk").read_bytes()
    v = np.ascontiguousarray(rng.standard_normal((dim, g.total)))
    S.write_vector_vtk(vdev(g, v), tmp_path / "c.vtk", "velocity")
    O.ref_lib().ref_write_vector_vtk(O.C.byref(g), O._ptr(v), str(tmp_path / "d.vtk").encode(), b"velocity")
    assert (tmp_path / "c.vtk").read_bytes() == (tmp_path / "d.vtk").read_bytes()


def test_new_entry_points_fail_like_the_reference():
    g2, g3 = S.make_grid(2, 4), S.make_grid(3, 3)
    with pytest.raises(ValueError):                 # problems.cpp:178: a 3D problem
        S.poisson3d_source(g2)
    with pytest.raises(ValueError):
        S.capacitor_sigma(g3, "medium")              # problems.cpp:504
    with pytest.raises(ValueError):
        S.trifoil_sources(g3, 0.2)                   # problems.cpp:386-389: leaves the unit domain
    with pytest.raises(ValueError):
        S.deformation_sources([[0.5, 0.5, 0.0], [0.5, 0.5, 0.0]], g2)   # zero-length curve
    with pytest.raises(OSError):
        S.write_field_vtk(S.Field(g3), "/nonexistent_dir/u.vtk", "u")  # io.cpp:17: io_error, cannot open
    f = S.Field(g3)
    bad = np.zeros(g3.total)
    bad[5] = np.nan
    probs = [S.ProblemSpec(g3, np.zeros(g3.total), bc=S.BoundarySpec.all_dirichlet(1.0)),
             S.ProblemSpec(g3, bad, bc=S.BoundarySpec.all_dirichlet(1.0))]
    with pytest.raises(ValueError):                 # cycle.cpp:150-152 inside the pipeline
        S.solve_many(probs, S.SolverConfig(tol=1e-10))
    # the context stays usable afterwards
    res = S.solve_many(probs[:1], S.SolverConfig(tol=1e-10))
    assert res[0].report.converged
