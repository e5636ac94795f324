"""The reference's OWN unit suites (proj/tests/unit/{grid,stencil,kernels,
cycle,problems,io}_tests.cpp, unmodified), compiled against this repo's
include/sgml headers with a doctest-compatible shim and linked with
libsgml_b200.so instead of proj/core (tests/cpp/Makefile ref-unit, built by
build() where /root/reference exists; the binary ships with the snapshot).
Every kernel-level and solve call in those suites runs on the B200.
oracle_tests.cpp is excluded: it needs Eigen and tests the reference's
direct-solver oracle, not the solve path."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_unit_tests")

pytestmark = pytest.mark.gpu


def test_reference_unit_suites_pass_against_the_b200_library(tmp_path):
    assert os.path.exists(BIN), "build/ref_unit_tests missing: run build() where /root/reference exists"
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900, cwd=tmp_path)
    print(out.stdout[-4000:], out.stderr[-4000:])
    assert out.returncode == 0, out.stderr[-4000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out.stdout)
    assert m and int(m.group(3)) == 0 and int(m.group(1)) == int(m.group(2)) >= 78
    # the binary really resolved the product library
    ldd = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libsgml_b200.so" in ldd and "sgml_ref" not in ldd
