"""ctypes binding of include/sgml_b200.h (the C-ABI of libsgml_b200.so).

The shared library is built in-tree (``paper_1703_07206_b200/lib``) by
``__graft_entry__.build()``.  There is no fallback: if the library is
missing or no CUDA device is present, compute entry points raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libsgml_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "sgml_b200.h")

OK, EINVAL, EBADSTEP, ENONFINITE, ECUDA, ENCCL, ELOGIC, EIO = range(8)


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int), ("N", C.c_int), ("pad_", C.c_int),
                ("h", C.c_double), ("total", C.c_uint64)]


class Bc(C.Structure):
    _fields_ = [("kind", C.c_int * 6), ("value", C.c_double * 6)]


class SolverCfg(C.Structure):
    _fields_ = [("n_r", C.c_int), ("max_cycles", C.c_int), ("tol", C.c_double),
                ("safety", C.c_double)]


class SolverOpts(C.Structure):
    _fields_ = [("engine", C.c_int), ("use_graph", C.c_int), ("timing", C.c_int),
                ("timing_classes", C.c_int), ("stencil", C.c_int), ("small_levels", C.c_int),
                ("cluster_levels", C.c_int), ("replicate_n", C.c_int)]


class CycleRecord(C.Structure):
    _fields_ = [("cycle", C.c_int), ("has_l1", C.c_int), ("work_units", C.c_uint64),
                ("residual", C.c_double), ("diag_min", C.c_double), ("l1_error", C.c_double)]


class DiagSample(C.Structure):
    _fields_ = [("cycle", C.c_int), ("pass_", C.c_int), ("level", C.c_int), ("pad_", C.c_int),
                ("value", C.c_double)]


HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_double))


class Report(C.Structure):
    _fields_ = [("rows", C.POINTER(CycleRecord)), ("rows_cap", C.c_int64), ("n_rows", C.c_int64),
                ("trace", C.POINTER(DiagSample)), ("trace_cap", C.c_int64), ("n_trace", C.c_int64),
                ("converged", C.c_int), ("nan_detected", C.c_int), ("stagnated", C.c_int),
                ("pad_", C.c_int), ("normalization", C.c_double), ("node_updates", C.c_uint64),
                ("hook", HOOK), ("hook_user", C.c_void_p), ("device_ms", C.c_double),
                ("kernel_launches", C.c_uint64), ("class_ms", C.c_double * 8),
                ("class_launches", C.c_uint64 * 8)]


CLASS_NAMES = ["relax0", "relax_coarse", "materialize", "pyramid", "residual", "literal", "other",
               "unused"]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_U64P = C.POINTER(C.c_uint64)

_SIGNATURES = {
    "sgml_last_error": ([], C.c_char_p),
    "sgml_version": ([], C.c_char_p),
    "sgml_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "sgml_ctx_create": ([C.c_int, C.POINTER(_P)], C.c_int),
    "sgml_ctx_destroy": ([_P], C.c_int),
    "sgml_ctx_synchronize": ([_P], C.c_int),
    "sgml_ctx_stream": ([_P], _P),
    "sgml_make_grid": ([C.c_int, C.c_int, C.POINTER(Grid)], C.c_int),
    "sgml_build_schedule": ([C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                             C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)], C.c_int),
    "sgml_closed_form_work_units": ([C.c_int, C.c_int], C.c_uint64),
    "sgml_field_create": ([_P, C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "sgml_field_destroy": ([_P], C.c_int),
    "sgml_field_upload": ([_P, _D], C.c_int),
    "sgml_field_download": ([_P, _D], C.c_int),
    "sgml_field_copy": ([_P, _P], C.c_int),
    "sgml_field_fill": ([_P, C.c_double], C.c_int),
    "sgml_field_grid": ([_P, C.POINTER(Grid)], C.c_int),
    "sgml_field_device_ptr": ([_P], _P),
    "sgml_restriction_into": ([_P, C.c_int, C.POINTER(Bc), _P, _P, _U64P], C.c_int),
    "sgml_relaxation_interpolation": ([_P, _P, _P, _P, C.c_int, _P, _P, C.c_double, C.c_double,
                                       C.POINTER(Bc), C.c_int, _D, _U64P], C.c_int),
    "sgml_residual_update": ([_P, _P, _P, C.c_double, C.POINTER(Bc)], C.c_int),
    "sgml_max_abs": ([_P, _D], C.c_int),
    "sgml_trapezoid_mean": ([_P, _D], C.c_int),
    "sgml_zero_mean_projection": ([_P], C.c_int),
    "sgml_apply_boundary": ([_P, C.POINTER(Bc), C.c_int], C.c_int),
    "sgml_restrict_sigma_levels": ([_P, C.POINTER(_P)], C.c_int),
    "sgml_pure_neumann_pin": ([_P], C.c_int),
    "sgml_single_cycle": ([_P, _P, _P, C.POINTER(_P), C.c_double, C.POINTER(Bc), C.c_int, C.c_int,
                           C.c_double, C.c_int, C.c_double, C.POINTER(SolverOpts), C.POINTER(Report),
                           _U64P], C.c_int),
    "sgml_single_cycle_state": ([_P, _P, _P, _P, _P, C.POINTER(C.c_int), _P, C.POINTER(_P), C.c_double,
                                 C.POINTER(Bc), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.c_int, C.c_double, C.c_int, C.c_double, C.POINTER(Report),
                                 _U64P], C.c_int),
    "sgml_solver_create": ([_P, C.c_int, C.c_int, C.POINTER(Bc), C.c_double, _P,
                            C.POINTER(SolverCfg), C.POINTER(SolverOpts), C.POINTER(_P)], C.c_int),
    "sgml_solver_destroy": ([_P], C.c_int),
    "sgml_solver_run": ([_P, _P, _P, C.POINTER(Report)], C.c_int),
    "sgml_solver_footprint": ([_P, _U64P], C.c_int),
    "sgml_solve": ([_P, C.c_int, C.c_int, C.POINTER(Bc), _D, _D, C.c_double, C.POINTER(SolverCfg),
                    C.POINTER(SolverOpts), _D, C.POINTER(Report)], C.c_int),
    "sgml_solve_many": ([_P, C.c_int, C.c_int, C.POINTER(Bc), C.c_int, C.POINTER(_D), _D, C.c_double,
                         C.POINTER(SolverCfg), C.POINTER(SolverOpts), C.POINTER(_D), C.POINTER(Report)], C.c_int),
    "sgml_nccl_unique_id": ([C.c_char_p], C.c_int),
    "sgml_ctx_join_nccl": ([_P, C.c_int, C.c_int, C.c_char_p], C.c_int),
    "sgml_local_group_create": ([C.c_int, C.POINTER(_P)], C.c_int),
    "sgml_local_group_destroy": ([_P], C.c_int),
    "sgml_ctx_join_local": ([_P, _P, C.c_int], C.c_int),
    "sgml_ctx_clique": ([_P, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "sgml_slab_plan_ex": ([C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                           C.POINTER(C.c_int)], C.c_int),
    "sgml_slab_plan": ([C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                        C.POINTER(C.c_int)], C.c_int),
    "sgml_axis_derivative": ([_P, C.c_int, _P], C.c_int),
    "sgml_gradient": ([_P, C.POINTER(_P)], C.c_int),
    "sgml_curl": ([C.POINTER(_P), C.POINTER(_P)], C.c_int),
    "sgml_divergence": ([C.POINTER(_P), _P], C.c_int),
    "sgml_deformation_velocity": ([_P, _P, C.c_double, C.c_double, C.POINTER(_P)], C.c_int),
    "sgml_move_nodes": ([_P, _P, C.c_double, C.c_double, C.c_int, C.POINTER(_P)], C.c_int),
    "sgml_sample_vector": ([C.POINTER(_P), C.c_int, _D, C.c_int, _D], C.c_int),
    "sgml_integrate_streamlines": ([C.POINTER(_P), _D, C.c_int, C.c_double, C.c_int, _D,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "sgml_build_poisson2d_source": ([_P], C.c_int),
    "sgml_build_poisson3d_source": ([_P], C.c_int),
    "sgml_build_sinsin2d_source": ([_P], C.c_int),
    "sgml_build_capacitor_sigma": ([_P, C.c_int], C.c_int),
    "sgml_build_trifoil_sources": ([C.POINTER(_P), C.c_double], C.c_int),
    "sgml_build_deformation_sources": ([_D, C.c_int, _P, _P, _D], C.c_int),
    "sgml_write_field_vtk": ([_P, C.c_char_p, C.c_char_p], C.c_int),
    "sgml_write_vector_vtk": ([C.POINTER(_P), C.c_char_p, C.c_char_p], C.c_int),
    "sgml_write_vtk_host": ([C.POINTER(_D), C.c_int, C.POINTER(Grid), C.c_char_p, C.c_char_p], C.c_int),
    "sgml_host_alloc": ([C.c_uint64, C.POINTER(_P)], C.c_int),
    "sgml_host_free": ([_P], C.c_int),
}

_lib = None


def header_symbols(path: str = HEADER_PATH) -> list[str]:
    """Every function name include/sgml_b200.h declares."""
    text = open(path).read()
    return sorted(set(re.findall(r"\b(sgml_[a-z0-9_]+)\s*\(", text)))


def lib() -> C.CDLL:
    """Load libsgml_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


class SgmlError(RuntimeError):
    """std::runtime_error analogue raised for CUDA / NCCL failures."""


class kernel_error(RuntimeError):  # noqa: N801 - mirrors sgml::kernel_error (kernels.hpp:38-40)
    """Raised when a kernel meets a non-finite value or a non-positive step."""


def check(status: int) -> None:
    if status == OK:
        return
    msg = (lib().sgml_last_error() or b"").decode()
    if status == EINVAL:
        raise ValueError(msg)
    if status in (EBADSTEP, ENONFINITE):
        raise kernel_error(msg)
    if status == ELOGIC:
        raise LookupError(msg)
    if status == EIO:
        raise OSError(msg)
    raise SgmlError(msg)


def device_count() -> int:
    c = C.c_int(0)
    check(lib().sgml_device_count(C.byref(c)))
    return c.value
