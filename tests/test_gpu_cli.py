"""The sgml_b200 command-line driver (tools/, the reference CLI's solve
subcommands on the device): its report.csv must carry the reference's
residual history bit for bit (%.17g round-trips doubles), its bench.csv the
reference's columns and work units."""
import csv
import os
import subprocess

import numpy as np
import pytest

from cases import O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "sgml_b200")


def run(args, out):
    p = subprocess.run([CLI] + args + ["--out", str(out)], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout + p.stderr


def report_rows(path):
    with open(path) as f:
        return [(int(r["cycle"]), int(r["work_units"]), float(r["residual"]), float(r["diag_residual_min"]))
                for r in csv.DictReader(f)]


def test_convergence_matches_the_oracle(tmp_path):
    rc, log = run(["convergence", "--n", "5", "--tol", "1e-10"], tmp_path)
    assert rc == 0, log
    g = O.make_grid(2, 5)
    ref = O.solve(g, O.all_dirichlet(0.0), O.fill("poisson2d", g), tol=1e-10, max_cycles=50)
    assert report_rows(tmp_path / "report.csv") == ref.rows
    with open(tmp_path / "trace.csv") as f:
        tr = [(int(r["cycle"]), int(r["pass"]), int(r["level"]), float(r["diag_residual"])) for r in csv.DictReader(f)]
    assert tr == ref.trace
    vals = open(tmp_path / "u.vtk").read().split("LOOKUP_TABLE default\n")[1].split()
    assert np.array_equal(np.array([float(v) for v in vals]), ref.u + 0.0)


@pytest.mark.parametrize("mode", ["high", "low"])
def test_capacitor_matches_the_oracle(tmp_path, mode):
    rc, log = run(["capacitor", "--n", "4", "--mode", mode, "--tol", "1e-10", "--no-vtk"], tmp_path)
    assert rc == 0, log
    g = O.make_grid(3, 4)
    s = O.fill("capacitor_sigma", g, -1.0 if mode == "high" else 1.0)
    b = O.make_bc([O.NEUMANN] * 4 + [O.DIRICHLET] * 2, [0.0] * 4 + [-1.0, 1.0])
    ref = O.solve(g, b, np.zeros(g.total), s, tol=1e-10, max_cycles=50)
    assert report_rows(tmp_path / "report.csv") == ref.rows


def test_bench_and_input_errors(tmp_path):
    rc, log = run(["bench", "--n", "6"], tmp_path)
    assert rc == 0, log
    with open(tmp_path / "bench.csv") as f:
        rows = list(csv.DictReader(f))
    assert [int(r["n"]) for r in rows] == [2, 3, 4, 5, 6]
    assert [int(r["work_units_per_cycle"]) for r in rows] == [O.closed_form_work_units(n, 2) for n in range(2, 7)]
    assert all(float(r["node_updates_per_second"]) > 0 for r in rows)
    assert run(["capacitor", "--mode", "medium"], tmp_path)[0] == 1
    assert run(["convergence", "--tol", "0"], tmp_path)[0] == 1
    # a budget too small to converge is reported with exit code 2
    assert run(["convergence", "--n", "5", "--tol", "1e-14", "--max-cycles", "2", "--no-vtk"], tmp_path)[0] == 2


def read_points(path):
    with open(path) as f:
        next(f)
        return np.array([[float(x) for x in line.split(",")] for line in f if line.strip()])


def vtk_values(path, kind):
    body = open(path).read().split(kind)[1].split("\n", 1)[1]
    if kind == "LOOKUP_TABLE default":
        return np.array([float(v) for v in body.split()])
    return np.array([float(v) for v in body.split()]).reshape(-1, 3)


def test_deform_matches_the_reference(tmp_path):
    # sgml_main.cpp:100-125 on the CLI smoke circle (32 points, r = 1/4)
    if O.ref_lib() is None:
        pytest.skip("deformation sources come from the reference build (oracle/_ref)")
    t = 2.0 * 3.14159265358979323846 * np.arange(32) / 32.0
    pts = np.stack([0.5 + 0.25 * np.cos(t), 0.5 + 0.25 * np.sin(t), np.zeros(32)], axis=1)
    curve = tmp_path / "circle.csv"
    curve.write_text("x,y\n" + "".join(f"{float(x)!r},{float(y)!r}\n" for x, y, _ in pts))
    rc, log = run(["deform", "--curve", str(curve), "--n", "5", "--a", "0.1", "--tol", "1e-10",
                   "--t", "0.5", "--steps", "8"], tmp_path)
    assert rc == 0, log
    g, f_raw, f, ri = O.ref_deformation_setup(pts, 0.1, 5)
    ref = O.solve(g, O.all_neumann(), f, a=0.1, tol=1e-10, max_cycles=50)
    assert report_rows(tmp_path / "report.csv") == ref.rows
    st, pos = O.move_nodes(g, ref.u, f_raw, ri, 0.5, 8)
    assert st == 0
    assert np.array_equal(read_points(tmp_path / "nodes.csv"), pos[:, :2] + 0.0)


def test_trifoil_matches_the_reference(tmp_path):
    # sgml_main.cpp:131-164: three potentials, v = curl psi, RK4 streamlines
    if O.ref_lib() is None:
        pytest.skip("trifoil sources come from the reference build (oracle/_ref)")
    rc, log = run(["trifoil", "--n", "4", "--tol", "1e-10", "--t", "0.01", "--steps", "300"], tmp_path)
    assert rc == 0, log
    us = []
    for c, name in zip("xyz", ("report.csv", "report_psi_y.csv", "report_psi_z.csv")):
        g, b, f, s, a = O.ref_problem("trifoil_" + c, 4)
        ref = O.solve(g, b, f, tol=1e-10, max_cycles=50)
        assert report_rows(tmp_path / name) == ref.rows
        us.append(ref.u)
    v = O.curl(g, np.stack(us))
    assert np.array_equal(vtk_values(tmp_path / "v.vtk", "VECTORS velocity double"), v.T + 0.0)
    for s, seed in enumerate(([0.5, 0.5, 0.5], [0.35, 0.5, 0.5])):
        pts, stop = O.integrate_streamline(g, v, seed, 0.01, 300)
        assert np.array_equal(read_points(tmp_path / f"streamline_{s}.csv"), pts + 0.0)


def test_capacitor_force_field(tmp_path):
    # sgml_main.cpp:166-178: F.vtk = gradient(u)
    rc, log = run(["capacitor", "--n", "3", "--mode", "low", "--tol", "1e-10"], tmp_path)
    assert rc == 0, log
    g = O.make_grid(3, 3)
    s = O.fill("capacitor_sigma", g, 1.0)
    b = O.make_bc([O.NEUMANN] * 4 + [O.DIRICHLET] * 2, [0.0] * 4 + [-1.0, 1.0])
    ref = O.solve(g, b, np.zeros(g.total), s, tol=1e-10, max_cycles=50)
    assert np.array_equal(vtk_values(tmp_path / "u.vtk", "LOOKUP_TABLE default"), ref.u + 0.0)
    assert np.array_equal(vtk_values(tmp_path / "F.vtk", "VECTORS F double"), np.vstack(
        [O.gradient(g, ref.u), np.zeros((0, g.total))]).T + 0.0)
