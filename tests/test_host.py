"""Host-side logic of the product library (no GPU needed).

Mirrors the schedule / work-unit rows of cycle_tests.cpp:16-67 and
grid_tests.cpp, and checks that libsgml_b200.so exports every symbol the
C-ABI header declares.
"""
import ctypes
import subprocess

import pytest

import paper_1703_07206_b200 as S
from paper_1703_07206_b200 import _capi


def test_library_exports_every_header_symbol():
    lib = _capi.lib()
    declared = _capi.header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    # and nm agrees (dynamic symbol table, defined text symbols)
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    for other in ("sm_90", "sm_80", "sm_103"):
        assert other not in out


def test_make_grid_matches_reference_rules():
    g = S.make_grid(3, 8)
    assert (g.N, g.total, g.h) == (257, 257 ** 3, 1.0 / 256)
    g2 = S.make_grid(2, 1)
    assert (g2.N, g2.total) == (3, 9)
    for dim, n in ((1, 3), (4, 3), (2, 0), (3, 14)):
        with pytest.raises(ValueError):
            S.make_grid(dim, n)


def test_schedule_n2_nr1_step_by_step():
    # cycle_tests.cpp:16-34
    s = S.build_schedule(2, 1)
    R, X = S.ScheduleStep.RESTRICT_SOURCE, S.ScheduleStep.RELAX
    assert [(st.kind, st.level, st.count) for st in s.steps] == [
        (R, 1, 1), (X, 1, 1), (R, 0, 1), (X, 0, 1), (R, 0, 1), (X, 0, 1), (X, 0, 1)]
    assert S.schedule_work_units(s) == 5


def test_schedule_counts_double_and_cap():
    # cycle_tests.cpp:36-45
    s = S.build_schedule(4, 8)
    lvl3 = [st.count for st in s.steps if st.kind == S.ScheduleStep.RELAX and st.level == 3]
    assert lvl3 == [2]
    assert s.steps[-1].count == 8 and s.steps[-1].level == 0


def test_frozen_work_unit_table():
    # cycle_tests.cpp:47-60 (+ the n = 9, 10, 11 values of SURVEY.md 3.2)
    table = {(2, 1): 5, (2, 2): 9, (2, 8): 13, (4, 1): 21, (4, 2): 32, (4, 8): 62, (6, 1): 57,
             (6, 2): 79, (6, 8): 155, (8, 1): 121, (8, 2): 158, (8, 8): 304, (7, 2): 114,
             (9, 2): 212, (10, 2): 277, (11, 2): 354}
    for (n, n_r), units in table.items():
        assert S.closed_form_work_units(n, n_r) == units


def test_closed_form_equals_enumeration():
    # cycle_tests.cpp:62-67
    for n in range(1, 11):
        for n_r in (1, 2, 3, 8):
            assert S.closed_form_work_units(n, n_r) == S.schedule_work_units(S.build_schedule(n, n_r))


def test_schedule_rejects_invalid_parameters():
    with pytest.raises(ValueError):
        S.build_schedule(0, 1)
    with pytest.raises(ValueError):
        S.build_schedule(3, 0)


def test_boundary_spec_tie_break_and_subsets():
    # grid_tests.cpp:96-105: lowest face id wins at corners
    bc = S.BoundarySpec.all_neumann()
    bc.set_face(0, 1, S.BcKind.dirichlet, 2.0)
    bc.set_face(1, 0, S.BcKind.dirichlet, 5.0)
    assert bc.dirichlet_value((4, 0, 0), 2, 5) == 2.0
    assert bc.on_dirichlet((4, 2), 2, 5) and not bc.on_dirichlet((0, 2), 2, 5)
    with pytest.raises(LookupError):
        bc.dirichlet_value((2, 2), 2, 5)
    assert S.in_level_subset((4, 8, 0), 2) and not S.in_level_subset((4, 6, 0), 2)
    assert [S.mirror_index(i, 5) for i in (-2, 0, 4, 6)] == [2, 0, 4, 2]
    with pytest.raises(IndexError):
        S.mirror_index(-5, 5)


def test_no_device_means_loud_failure():
    if S.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises((S.SgmlError, ValueError)):
        S.Context(0)


def test_c_abi_struct_layouts():
    assert ctypes.sizeof(_capi.Grid) == 32
    assert ctypes.sizeof(_capi.Bc) == 72
    assert ctypes.sizeof(_capi.CycleRecord) == 40
    assert ctypes.sizeof(_capi.DiagSample) == 24


def test_c_abi_struct_sizes_match_the_header(tmp_path):
    # the ctypes mirrors (paper_1703_07206_b200/_capi.py) against the C compiler's
    # view of include/sgml_b200.h
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include "sgml_b200.h"\nint main(void) {\n'
                   'printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(sgml_grid), sizeof(sgml_bc), '
                   'sizeof(sgml_solver_cfg), sizeof(sgml_solver_opts), sizeof(sgml_cycle_record), '
                   'sizeof(sgml_diag_sample), sizeof(sgml_report));\nreturn 0; }\n')
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(t) for t in (_capi.Grid, _capi.Bc, _capi.SolverCfg, _capi.SolverOpts,
                                       _capi.CycleRecord, _capi.DiagSample, _capi.Report)]
    assert got == want
