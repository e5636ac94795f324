"""ctypes view of the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``C``   — oracle/_build/libsgml_oracle.so, the C restatement of the
  reference solve path (oracle/sgml_oracle.c).  Builds anywhere.
* ``REF`` — oracle/_ref/libsgml_ref.so, the UNMODIFIED reference core compiled
  in place from /root/reference (oracle/Makefile ``ref``), or None when that
  tree was not available at build time.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(paper_1703_07206_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB_PATH = os.path.join(HERE, "_build", "libsgml_oracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libsgml_ref.so")
REF_SOURCE = "/root/reference/proj/core"

DIRICHLET, NEUMANN = 0, 1


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int), ("N", C.c_int), ("pad_", C.c_int),
                ("h", C.c_double), ("total", C.c_uint64)]


class Bc(C.Structure):
    _fields_ = [("kind", C.c_int * 6), ("value", C.c_double * 6)]


class Row(C.Structure):
    _fields_ = [("cycle", C.c_int), ("pad_", C.c_int), ("work_units", C.c_uint64),
                ("residual", C.c_double), ("diag_min", C.c_double)]


class Sample(C.Structure):
    _fields_ = [("cycle", C.c_int), ("pass_", C.c_int), ("level", C.c_int), ("pad_", C.c_int),
                ("value", C.c_double)]


class Report(C.Structure):
    _fields_ = [("rows", C.POINTER(Row)), ("rows_cap", C.c_int64), ("n_rows", C.c_int64),
                ("trace", C.POINTER(Sample)), ("trace_cap", C.c_int64), ("n_trace", C.c_int64),
                ("converged", C.c_int), ("nan_detected", C.c_int), ("stagnated", C.c_int),
                ("pad_", C.c_int), ("normalization", C.c_double), ("node_updates", C.c_uint64)]


def build(with_ref: bool | None = None) -> None:
    """Compile the C restatement (and the reference when its tree exists)."""
    subprocess.check_call(["make", "-s", "-C", HERE], stdout=subprocess.DEVNULL)
    if with_ref is None:
        with_ref = os.path.isdir(REF_SOURCE)
    if with_ref:
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"], stdout=subprocess.DEVNULL)


_D = C.POINTER(C.c_double)
_U64P = C.POINTER(C.c_uint64)


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _load_c():
    if not os.path.exists(C_LIB_PATH):
        build(with_ref=False)
    lib = C.CDLL(C_LIB_PATH)
    G, B = C.POINTER(Grid), C.POINTER(Bc)
    lib.og_make_grid.argtypes = [C.c_int, C.c_int, G]
    lib.og_restrict_pass.argtypes = [G, B, _D, _D, C.c_int]
    lib.og_restriction_into.argtypes = [G, B, _D, C.c_int, _D, _D, _U64P]
    lib.og_relaxation_interpolation.argtypes = [G, B, _D, _D, _D, _D, C.c_int, _D, _D, C.c_double,
                                                C.c_double, C.c_int, _D, _U64P]
    lib.og_residual_update.argtypes = [G, B, _D, _D, _D, C.c_double]
    lib.og_apply_operator.argtypes = [G, B, _D, _D, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int]
    lib.og_apply_operator.restype = C.c_double
    lib.og_max_abs.argtypes = [_D, C.c_uint64]
    lib.og_max_abs.restype = C.c_double
    lib.og_trapezoid_mean.argtypes = [G, _D]
    lib.og_trapezoid_mean.restype = C.c_double
    lib.og_zero_mean_projection.argtypes = [G, _D]
    lib.og_apply_boundary.argtypes = [G, B, _D, C.c_int]
    lib.og_build_schedule.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.c_int]
    lib.og_closed_form_work_units.argtypes = [C.c_int, C.c_int]
    lib.og_closed_form_work_units.restype = C.c_uint64
    lib.og_restrict_sigma_levels.argtypes = [G, _D, _D]
    lib.og_single_cycle.argtypes = [G, B, _D, _D, _D, _D, _D, _D, C.c_double, C.c_int, C.c_int,
                                    C.c_double, C.c_int, C.c_double, C.POINTER(Report), _U64P]
    lib.og_solve.argtypes = [G, B, _D, _D, C.c_double, C.c_int, C.c_double, C.c_int, C.c_double,
                             _D, C.POINTER(Report)]
    for fn in ("og_fill_poisson2d", "og_fill_poisson3d", "og_fill_sinsin2d"):
        getattr(lib, fn).argtypes = [G, _D]
    lib.og_fill_capacitor_sigma.argtypes = [G, C.c_double, _D]
    lib.og_lcg_fill.argtypes = [_D, C.c_uint64, C.c_uint64]
    lib.og_set_stencil.argtypes = [C.c_int]
    lib.og_get_stencil.restype = C.c_int
    lib.og_axis_derivative.argtypes = [G, _D, C.c_int, _D]
    for fn in ("og_gradient", "og_curl", "og_divergence"):
        getattr(lib, fn).argtypes = [G, _D, _D]
    lib.og_deformation_velocity.argtypes = [G, _D, _D, C.c_double, C.c_double, _D]
    lib.og_move_nodes.argtypes = [G, _D, _D, C.c_double, C.c_double, C.c_int, _D]
    lib.og_sample_vector.argtypes = [G, _D, C.c_int, _D, _D]
    lib.og_integrate_streamline.argtypes = [G, _D, _D, C.c_double, C.c_int, _D, C.POINTER(C.c_int)]
    return lib


def _load_ref():
    if not os.path.exists(REF_LIB_PATH):
        if not os.path.isdir(REF_SOURCE):
            return None
        build(with_ref=True)
    lib = C.CDLL(REF_LIB_PATH)
    G, B = C.POINTER(Grid), C.POINTER(Bc)
    lib.ref_restriction_into.argtypes = [G, B, _D, C.c_int, _D, _U64P]
    lib.ref_relaxation_interpolation.argtypes = [G, B, _D, _D, _D, _D, C.c_int, _D, _D, C.c_double,
                                                 C.c_double, C.c_int, _D, _U64P]
    lib.ref_residual_update.argtypes = [G, B, _D, _D, _D, C.c_double]
    lib.ref_max_abs.argtypes = [G, _D]
    lib.ref_max_abs.restype = C.c_double
    lib.ref_trapezoid_mean.argtypes = [G, _D]
    lib.ref_trapezoid_mean.restype = C.c_double
    lib.ref_closed_form_work_units.argtypes = [C.c_int, C.c_int]
    lib.ref_closed_form_work_units.restype = C.c_uint64
    lib.ref_single_cycle.argtypes = [G, B, _D, _D, _D, C.c_double, C.c_int, C.c_int, C.c_double,
                                     C.c_int, C.c_double, C.POINTER(Report), _U64P]
    lib.ref_solve.argtypes = [G, B, _D, _D, C.c_double, C.c_int, C.c_double, C.c_int, C.c_double,
                              _D, C.POINTER(Report)]
    lib.ref_problem_fields.argtypes = [C.c_char_p, C.c_int, _D, _D, C.POINTER(C.c_int), _D, _D]
    for fn in ("ref_gradient", "ref_curl", "ref_divergence"):
        getattr(lib, fn).argtypes = [G, _D, _D]
    lib.ref_deformation_velocity.argtypes = [G, _D, _D, C.c_double, C.c_double, _D]
    lib.ref_move_nodes.argtypes = [G, _D, _D, C.c_double, C.c_double, C.c_int, _D]
    lib.ref_sample_vector.argtypes = [G, _D, _D, _D]
    lib.ref_integrate_streamline.argtypes = [G, _D, _D, C.c_double, C.c_int, _D, C.POINTER(C.c_int)]
    lib.ref_deformation_setup.argtypes = [_D, C.c_int, C.c_double, C.c_int, _D, _D, _D]
    lib.ref_write_field_vtk.argtypes = [G, _D, C.c_char_p, C.c_char_p]
    lib.ref_write_vector_vtk.argtypes = [G, _D, C.c_char_p, C.c_char_p]
    lib.ref_single_cycle_state.argtypes = [G, B, _D, _D, _D, _D, C.POINTER(C.c_int), _D, _D, C.c_int, C.c_double,
                                           C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                           C.c_int, C.c_double, C.c_int, C.c_double, C.POINTER(Report), _U64P]
    lib.ref_session_create.argtypes = [G, B, _D, _D, C.c_double, C.c_int, C.c_double]
    lib.ref_session_create.restype = C.c_void_p
    lib.ref_session_destroy.argtypes = [C.c_void_p]
    lib.ref_session_nsteps.argtypes = [C.c_void_p]
    lib.ref_session_begin_cycle.argtypes = [C.c_void_p, C.c_int]
    lib.ref_session_step.argtypes = [C.c_void_p, C.c_int, _D]
    lib.ref_session_recurrence.argtypes = [C.c_void_p]
    lib.ref_session_recurrence.restype = C.c_double
    return lib


_c_lib = None
_ref_lib = None
_ref_probed = False


def c_lib():
    global _c_lib
    if _c_lib is None:
        _c_lib = _load_c()
    return _c_lib


def ref_lib():
    """The compiled reference, or None when it is unavailable on this host."""
    global _ref_lib, _ref_probed
    if not _ref_probed:
        _ref_probed = True
        _ref_lib = _load_ref()
    return _ref_lib


# ------------------------------------------------------------ helpers ----

def make_grid(dim: int, n: int) -> Grid:
    g = Grid()
    if c_lib().og_make_grid(dim, n, C.byref(g)) != 0:
        raise ValueError("make_grid: dim must be 2 or 3 and n in [1, 13]")
    return g


def make_bc(kinds, values=None) -> Bc:
    b = Bc()
    values = values if values is not None else [0.0] * 6
    for f in range(6):
        b.kind[f] = int(kinds[f])
        b.value[f] = float(values[f])
    return b


def all_dirichlet(value=0.0) -> Bc:
    return make_bc([DIRICHLET] * 6, [value] * 6)


def all_neumann() -> Bc:
    return make_bc([NEUMANN] * 6)


def shape_of(g: Grid):
    return (g.N,) * g.dim


def lcg(g_or_total, seed: int) -> np.ndarray:
    total = g_or_total.total if isinstance(g_or_total, Grid) else int(g_or_total)
    out = np.empty(total, np.float64)
    c_lib().og_lcg_fill(_ptr(out), total, seed)
    return out


@dataclass
class SolveOut:
    u: np.ndarray
    rows: list = field(default_factory=list)        # (cycle, work_units, residual, diag_min)
    trace: list = field(default_factory=list)       # (cycle, pass, level, value)
    converged: bool = False
    nan_detected: bool = False
    stagnated: bool = False
    normalization: float = 0.0
    node_updates: int = 0
    status: int = 0


def _report(rows_cap=4096, trace_cap=1 << 20):
    rows = (Row * rows_cap)()
    trace = (Sample * trace_cap)()
    rep = Report()
    rep.rows, rep.rows_cap = C.cast(rows, C.POINTER(Row)), rows_cap
    rep.trace, rep.trace_cap = C.cast(trace, C.POINTER(Sample)), trace_cap
    return rep, rows, trace


def _collect(u, rep, rows, trace, status) -> SolveOut:
    out = SolveOut(u=u, status=status)
    out.rows = [(rows[i].cycle, rows[i].work_units, rows[i].residual, rows[i].diag_min)
                for i in range(min(rep.n_rows, rep.rows_cap))]
    out.trace = [(trace[i].cycle, trace[i].pass_, trace[i].level, trace[i].value)
                 for i in range(min(rep.n_trace, rep.trace_cap))]
    out.converged, out.nan_detected, out.stagnated = bool(rep.converged), bool(rep.nan_detected), \
        bool(rep.stagnated)
    out.normalization, out.node_updates = rep.normalization, rep.node_updates
    return out


def solve(g: Grid, bc: Bc, f, sigma=None, a=0.0, n_r=2, tol=1e-12, max_cycles=50, safety=0.9,
          impl: str = "c") -> SolveOut:
    """Run the oracle solve ('c' restatement or 'ref' compiled reference)."""
    u = np.zeros(g.total, np.float64)
    rep, rows, trace = _report()
    f = np.ascontiguousarray(f, np.float64).reshape(-1)
    sig = None if sigma is None else np.ascontiguousarray(sigma, np.float64).reshape(-1)
    if impl == "c":
        st = c_lib().og_solve(C.byref(g), C.byref(bc), _ptr(f), _ptr(sig), a, n_r, tol,
                              max_cycles, safety, _ptr(u), C.byref(rep))
    else:
        st = ref_lib().ref_solve(C.byref(g), C.byref(bc), _ptr(f), _ptr(sig), a, n_r, tol,
                                 max_cycles, safety, _ptr(u), C.byref(rep))
    return _collect(u, rep, rows, trace, st)


def relax(g: Grid, bc: Bc, u_prev, du_prev, level, gsrc, sigma=None, a=0.0, safety=0.9,
          homogeneous=False, impl: str = "c"):
    """One relaxation-interpolation pass; returns (status, u, du, diag)."""
    u = np.zeros(g.total, np.float64)
    du = np.zeros(g.total, np.float64)
    diag = C.c_double(0.0)
    work = C.c_uint64(0)
    args = (C.byref(g), C.byref(bc), _ptr(u), _ptr(u_prev), _ptr(du), _ptr(du_prev), level,
            _ptr(gsrc), _ptr(sigma), a, safety, int(homogeneous), C.byref(diag), C.byref(work))
    fn = c_lib().og_relaxation_interpolation if impl == "c" else ref_lib().ref_relaxation_interpolation
    st = fn(*args)
    return st, u, du, diag.value


def restriction(g: Grid, bc: Bc, f, v, impl: str = "c"):
    out = np.zeros(g.total, np.float64)
    work = C.c_uint64(0)
    if impl == "c":
        scratch = np.zeros(g.total, np.float64)
        c_lib().og_restriction_into(C.byref(g), C.byref(bc), _ptr(f), v, _ptr(out), _ptr(scratch),
                                    C.byref(work))
    else:
        ref_lib().ref_restriction_into(C.byref(g), C.byref(bc), _ptr(f), v, _ptr(out), C.byref(work))
    return out, work.value


def residual_update(g: Grid, bc: Bc, r, e, sigma=None, a=0.0, impl: str = "c"):
    r = np.array(r, np.float64, copy=True)
    fn = c_lib().og_residual_update if impl == "c" else ref_lib().ref_residual_update
    fn(C.byref(g), C.byref(bc), _ptr(r), _ptr(e), _ptr(sigma), a)
    return r


def single_cycle(g: Grid, bc: Bc, source, sigma_levels=None, a=0.0, homogeneous=False, n_r=2,
                 safety=0.9, cycle_index=0, normalization=1.0, impl: str = "c"):
    """Returns (status, state.u, trace, work) of one cycle from the zero state."""
    T = g.total
    u = np.zeros(T, np.float64)
    rep, rows, trace = _report()
    work = C.c_uint64(0)
    sl = None if sigma_levels is None else np.ascontiguousarray(sigma_levels, np.float64).reshape(-1)
    if impl == "c":
        up = np.zeros(T, np.float64)
        du = np.zeros(T, np.float64)
        dup = np.zeros(T, np.float64)
        st = c_lib().og_single_cycle(C.byref(g), C.byref(bc), _ptr(u), _ptr(up), _ptr(du), _ptr(dup),
                                     _ptr(source), _ptr(sl), a, int(homogeneous), n_r, safety,
                                     cycle_index, normalization, C.byref(rep), C.byref(work))
    else:
        st = ref_lib().ref_single_cycle(C.byref(g), C.byref(bc), _ptr(u), _ptr(source), _ptr(sl), a,
                                        int(homogeneous), n_r, safety, cycle_index, normalization,
                                        C.byref(rep), C.byref(work))
    out = _collect(u, rep, rows, trace, st)
    return st, u, out.trace, work.value


def sigma_levels(g: Grid, sigma) -> np.ndarray:
    out = np.zeros(g.n * g.total, np.float64)
    st = c_lib().og_restrict_sigma_levels(C.byref(g), _ptr(np.ascontiguousarray(sigma)), _ptr(out))
    if st != 0:
        raise ValueError("restrict_sigma_levels: coefficient must stay positive")
    return out


def fill(name: str, g: Grid, sign: float = 1.0) -> np.ndarray:
    out = np.zeros(g.total, np.float64)
    lib = c_lib()
    if name == "capacitor_sigma":
        lib.og_fill_capacitor_sigma(C.byref(g), sign, _ptr(out))
    else:
        getattr(lib, "og_fill_" + name)(C.byref(g), _ptr(out))
    return out


def ref_problem(name: str, n: int):
    """(grid, bc, f, sigma|None, a) exactly as the reference's builders make them."""
    lib = ref_lib()
    if lib is None:
        raise RuntimeError("reference build unavailable")
    dim = 2 if name in ("poisson2d", "deformation_circle") else 3
    g = make_grid(dim, n)
    f = np.zeros(g.total, np.float64)
    sig = np.zeros(g.total, np.float64)
    kinds = (C.c_int * 6)()
    vals = (C.c_double * 6)()
    a = C.c_double(0.0)
    rc = lib.ref_problem_fields(name.encode(), n, _ptr(f), _ptr(sig), kinds, vals, C.byref(a))
    if rc not in (2, 3):
        raise ValueError(name)
    bc = make_bc(list(kinds), list(vals))
    return g, bc, f, (sig if rc == 3 else None), a.value


def ref_single_cycle_state(g: Grid, bc: Bc, u, u_prev, du, du_prev, level, source, sigma_levels, a, homogeneous,
                           steps, safety, cycle_index, normalization, work=0):
    """The reference's single_cycle on an arbitrary state / schedule / sigma
    levels; returns (status, u, u_prev, du, du_prev, level, trace, work)."""
    lib = ref_lib()
    arrs = [np.ascontiguousarray(x, np.float64).reshape(-1).copy() for x in (u, u_prev, du, du_prev)]
    lv = None if sigma_levels is None else np.ascontiguousarray(sigma_levels, np.float64).reshape(-1)
    nl = 0 if sigma_levels is None else len(sigma_levels)
    n = len(steps)
    kinds = (C.c_int * max(n, 1))(*[s[0] for s in steps])
    levels = (C.c_int * max(n, 1))(*[s[1] for s in steps])
    counts = (C.c_int * max(n, 1))(*[s[2] for s in steps])
    lev = C.c_int(level)
    w = C.c_uint64(work)
    rep, rows, trace = _report()
    src = np.ascontiguousarray(source, np.float64).reshape(-1)
    st = lib.ref_single_cycle_state(C.byref(g), C.byref(bc), *[_ptr(x) for x in arrs], C.byref(lev), _ptr(src),
                                    _ptr(lv), nl, a, int(homogeneous), kinds, levels, counts, n, safety, cycle_index,
                                    normalization, C.byref(rep), C.byref(w))
    tr = [(trace[i].cycle, trace[i].pass_, trace[i].level, trace[i].value)
          for i in range(min(rep.n_trace, rep.trace_cap))]
    return st, arrs[0], arrs[1], arrs[2], arrs[3], lev.value, tr, w.value


class RefSession:
    """The reference's solve driven one schedule step at a time (timing only:
    bench.py's reference arm and cpu_baseline; oracle/ref_shim.cpp)."""

    def __init__(self, g: Grid, bc: Bc, f, sigma=None, a=0.0, n_r=2, safety=0.9):
        lib = ref_lib()
        if lib is None:
            raise RuntimeError("reference build unavailable")
        self.lib = lib
        f = np.ascontiguousarray(f, np.float64).reshape(-1)
        sig = None if sigma is None else np.ascontiguousarray(sigma, np.float64).reshape(-1)
        self.h = lib.ref_session_create(C.byref(g), C.byref(bc), _ptr(f), _ptr(sig), a, n_r, safety)
        self.schedule = build_schedule(g.n, n_r)
        assert lib.ref_session_nsteps(self.h) == len(self.schedule)

    @staticmethod
    def units(step) -> int:
        kind, level, count = step
        return level if kind == 0 else count

    def begin_cycle(self, homogeneous: bool = False) -> None:
        self.lib.ref_session_begin_cycle(self.h, int(homogeneous))

    def step(self, index: int) -> int:
        d = np.zeros(1)
        return self.lib.ref_session_step(self.h, index, _ptr(d))

    def recurrence(self) -> float:
        return self.lib.ref_session_recurrence(self.h)

    def close(self) -> None:
        if self.h:
            self.lib.ref_session_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def closed_form_work_units(n: int, n_r: int) -> int:
    return int(c_lib().og_closed_form_work_units(n, n_r))


def build_schedule(n: int, n_r: int):
    cap = 4096
    k = (C.c_int * cap)()
    lv = (C.c_int * cap)()
    cn = (C.c_int * cap)()
    c = c_lib().og_build_schedule(n, n_r, k, lv, cn, cap)
    if c < 0:
        raise ValueError("build_schedule: n and n_r must be >= 1")
    return [(k[i], lv[i], cn[i]) for i in range(c)]


# ------------------------------------------------- post-solve fields ----
# problems.cpp:40-97, 327-455.  Vector fields: (ncomp, total) arrays.
# impl "c" = the restatement, "ref" = the reference build (oracle/_ref).

def _lib(impl):
    lib = c_lib() if impl == "c" else ref_lib()
    if lib is None:
        raise RuntimeError("reference build unavailable")
    return lib, ("og_" if impl == "c" else "ref_")


def axis_derivative(g: Grid, u, axis: int):
    out = np.zeros(g.total)
    c_lib().og_axis_derivative(C.byref(g), _ptr(u), axis, _ptr(out))
    return out


def gradient(g: Grid, u, impl: str = "c"):
    lib, pre = _lib(impl)
    out = np.zeros((g.dim, g.total))
    getattr(lib, pre + "gradient")(C.byref(g), _ptr(u), _ptr(out))
    return out


def curl(g: Grid, psi, impl: str = "c"):
    lib, pre = _lib(impl)
    psi = np.ascontiguousarray(psi, np.float64)
    out = np.zeros((3, g.total))
    getattr(lib, pre + "curl")(C.byref(g), _ptr(psi), _ptr(out))
    return out


def divergence(g: Grid, v, impl: str = "c"):
    lib, pre = _lib(impl)
    v = np.ascontiguousarray(v[:g.dim], np.float64)
    out = np.zeros(g.total)
    getattr(lib, pre + "divergence")(C.byref(g), _ptr(v), _ptr(out))
    return out


def deformation_velocity(g: Grid, u, f_raw, raw_integral: float, t: float, impl: str = "c"):
    """(status, velocity (dim, total)); status 1 = zero denominator (invalid_argument)."""
    lib, pre = _lib(impl)
    out = np.zeros((g.dim, g.total))
    st = getattr(lib, pre + "deformation_velocity")(C.byref(g), _ptr(u), _ptr(f_raw), raw_integral, t, _ptr(out))
    return st, out


def move_nodes(g: Grid, u, f_raw, raw_integral: float, t: float, steps: int, impl: str = "c"):
    """(status, positions (total, 3))."""
    lib, pre = _lib(impl)
    pos = np.zeros((g.total, 3))
    st = getattr(lib, pre + "move_nodes")(C.byref(g), _ptr(u), _ptr(f_raw), raw_integral, t, steps, _ptr(pos))
    return st, pos


def sample_vector(g: Grid, v, pt, impl: str = "c"):
    v = np.ascontiguousarray(v[:g.dim], np.float64)
    p = np.ascontiguousarray(pt, np.float64)
    out = np.zeros(3)
    if impl == "c":
        c_lib().og_sample_vector(C.byref(g), _ptr(v), g.dim, _ptr(p), _ptr(out))
    else:
        ref_lib().ref_sample_vector(C.byref(g), _ptr(v), _ptr(p), _ptr(out))
    return out


def integrate_streamline(g: Grid, v, seed, step: float, max_steps: int, impl: str = "c"):
    """(points (count, 3), stop) with stop 0 max_steps, 1 left_domain, 2 stagnation."""
    lib, pre = _lib(impl)
    v = np.ascontiguousarray(v[:g.dim], np.float64)
    sd = np.ascontiguousarray(seed, np.float64)
    pts = np.zeros((max_steps + 1, 3))
    stop = C.c_int(0)
    cnt = getattr(lib, pre + "integrate_streamline")(C.byref(g), _ptr(v), _ptr(sd), step, max_steps, _ptr(pts),
                                                     C.byref(stop))
    return pts[:cnt].copy(), stop.value


def ref_deformation_setup(points, a: float, n: int):
    """deformation_problem of the reference for a closed curve: (grid, f_raw, f, raw_integral)."""
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    dim = 3 if np.any(pts[:, 2] != 0.0) else 2
    g = make_grid(dim, n)
    f_raw = np.zeros(g.total)
    f = np.zeros(g.total)
    ri = C.c_double(0.0)
    ref_lib().ref_deformation_setup(_ptr(pts), pts.shape[0], a, n, _ptr(f_raw), _ptr(f), C.byref(ri))
    return g, f_raw, f, ri.value


# ------------------------------------------------------ stencil family ----

class stencil:
    """Context manager: run the C restatement with stencil family `mode`
    (0 radial = the reference's, 1 compact 5/7-point, SURVEY.md 8a row a23,
    parity unpinned)."""

    def __init__(self, mode):
        self.mode = 1 if mode in (1, "compact") else 0

    def __enter__(self):
        self.prev = c_lib().og_get_stencil()
        c_lib().og_set_stencil(self.mode)
        return self

    def __exit__(self, *exc):
        c_lib().og_set_stencil(self.prev)
        return False
