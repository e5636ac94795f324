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
