"""The drop-in C++ API (include/sgml/*.hpp over libsgml_b200.so), driven by
tests/cpp/test_dropin.cpp the way the reference's C++ unit tests drive
proj/core, with bit-parity checks against the oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_dropin")

pytestmark = pytest.mark.gpu


def test_cpp_dropin_api():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 6
