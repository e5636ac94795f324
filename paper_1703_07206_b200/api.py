"""Python mirror of the reference C++ solver API (proj/core/include/sgml).

Same names, argument meaning and error behaviour as the reference:
``std::invalid_argument`` -> ``ValueError``, ``sgml::kernel_error`` ->
``kernel_error``.  Every compute call goes through the C-ABI of
``libsgml_b200.so`` (include/sgml_b200.h) onto the B200; fields passed to
the kernel-level functions are device-resident (:class:`Field`).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import check, kernel_error, lib

__all__ = [
    "BcKind", "FaceBc", "BoundarySpec", "Grid", "make_grid", "in_level_subset", "mirror_index",
    "Context", "default_context", "Field", "SolveState", "OperatorCoefficients",
    "restriction", "restriction_into", "relaxation_interpolation", "residual", "residual_update",
    "max_abs", "trapezoid_mean", "zero_mean_projection", "apply_boundary", "ScheduleStep",
    "CycleSchedule", "build_schedule", "closed_form_work_units", "schedule_work_units",
    "SolverConfig", "SolverOptions", "DiagSample", "CycleRecord", "SolveReport", "ProblemSpec",
    "SolveResult", "single_cycle", "single_cycle_state", "solve", "solve_many", "Solver", "restrict_sigma_levels", "pure_neumann_pin",
    "kernel_error", "LocalGroup", "nccl_unique_id", "slab_plan",
]


# ---------------------------------------------------------------- grid ----

class BcKind(enum.IntEnum):
    """grid.hpp:121-124"""
    dirichlet = 0
    neumann = 1


@dataclass
class FaceBc:
    kind: BcKind = BcKind.dirichlet
    value: float = 0.0


@dataclass
class BoundarySpec:
    """grid.hpp:125-157: six faces, id = axis*2 + side."""
    faces: list = field(default_factory=lambda: [FaceBc() for _ in range(6)])

    @staticmethod
    def face_id(axis: int, side: int) -> int:
        return axis * 2 + side

    def face(self, axis: int, side: int) -> FaceBc:
        return self.faces[axis * 2 + side]

    def set_face(self, axis: int, side: int, kind: BcKind, value: float = 0.0) -> None:
        self.faces[axis * 2 + side] = FaceBc(BcKind(kind), float(value))

    @staticmethod
    def all_dirichlet(value: float = 0.0) -> "BoundarySpec":
        return BoundarySpec([FaceBc(BcKind.dirichlet, float(value)) for _ in range(6)])

    @staticmethod
    def all_neumann() -> "BoundarySpec":
        return BoundarySpec([FaceBc(BcKind.neumann, 0.0) for _ in range(6)])

    def any_dirichlet(self, dim: int) -> bool:
        return any(self.faces[f].kind == BcKind.dirichlet for f in range(2 * dim))

    def all_faces_neumann(self, dim: int) -> bool:
        return not self.any_dirichlet(dim)

    def on_dirichlet(self, idx, dim: int, N: int) -> bool:
        c = tuple(idx) + (0,) * (3 - len(tuple(idx)))
        for a in range(dim):
            if c[a] == 0 and self.faces[2 * a].kind == BcKind.dirichlet:
                return True
            if c[a] == N - 1 and self.faces[2 * a + 1].kind == BcKind.dirichlet:
                return True
        return False

    def dirichlet_value(self, idx, dim: int, N: int) -> float:
        c = tuple(idx) + (0,) * (3 - len(tuple(idx)))
        for a in range(dim):
            if c[a] == 0 and self.faces[2 * a].kind == BcKind.dirichlet:
                return self.faces[2 * a].value
            if c[a] == N - 1 and self.faces[2 * a + 1].kind == BcKind.dirichlet:
                return self.faces[2 * a + 1].value
        raise LookupError("dirichlet_value: node is not on a Dirichlet face")

    def to_c(self) -> _capi.Bc:
        b = _capi.Bc()
        for f in range(6):
            b.kind[f] = int(self.faces[f].kind)
            b.value[f] = float(self.faces[f].value)
        return b


@dataclass(frozen=True)
class Grid:
    """grid.hpp:31-39"""
    dim: int = 2
    n: int = 1
    N: int = 3
    h: float = 0.5
    total: int = 9

    @property
    def shape(self):
        """numpy shape of a field in the reference's x-fastest order."""
        return (self.N,) * self.dim


def make_grid(dim: int, n: int) -> Grid:
    """grid.cpp:10-23 (ValueError outside dim in {2,3}, n in [1,13])."""
    g = _capi.Grid()
    check(lib().sgml_make_grid(dim, n, C.byref(g)))
    return Grid(g.dim, g.n, g.N, g.h, int(g.total))


def in_level_subset(idx, v: int) -> bool:
    """grid.hpp:54-57"""
    mask = (1 << v) - 1
    i, j, k = (tuple(idx) + (0, 0, 0))[:3]
    return ((i | j | k) & mask) == 0


def mirror_index(i: int, N: int) -> int:
    """grid.hpp:63-69"""
    if i < 0:
        i = -i
    elif i > N - 1:
        i = 2 * (N - 1) - i
    if i < 0 or i > N - 1:
        raise IndexError("mirror_index: reflection still out of range")
    return i


# ------------------------------------------------------------- context ----

class Context:
    """One CUDA device + one stream (sgml_ctx)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().sgml_ctx_create(device, C.byref(self._h)))
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        """cudaStream_t of this context (every kernel launches on it)."""
        return int(lib().sgml_ctx_stream(self._h) or 0)

    def synchronize(self) -> None:
        check(lib().sgml_ctx_synchronize(self._h))

    # ---- multi-GPU clique (z-slab solves) ------------------
    def join_nccl(self, nranks: int, rank: int, unique_id: bytes) -> None:
        """Join an NCCL clique (one process per GPU); rank 0 makes the id
        with nccl_unique_id() and shares it (e.g. torch.distributed)."""
        if len(unique_id) != 128:
            raise ValueError("join_nccl: the NCCL unique id is 128 bytes")
        check(lib().sgml_ctx_join_nccl(self._h, nranks, rank, unique_id))

    def join_local(self, group: "LocalGroup", rank: int) -> None:
        """Join an in-process clique (one host thread per rank)."""
        check(lib().sgml_ctx_join_local(self._h, group.handle, rank))
        self._group = group  # keep the group alive

    def clique(self) -> tuple[int, int]:
        """(nranks, rank) of the clique this context belongs to."""
        n, r = C.c_int(), C.c_int()
        check(lib().sgml_ctx_clique(self._h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def close(self) -> None:
        if self._h:
            lib().sgml_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """In-process clique of `nranks` ranks (one host thread per rank; the
    decomposition's parity tests run it on one GPU)."""

    def __init__(self, nranks: int):
        self._h = C.c_void_p()
        check(lib().sgml_local_group_create(nranks, C.byref(self._h)))
        self.nranks = nranks

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                lib().sgml_local_group_destroy(self._h)
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """A new NCCL clique id (128 bytes) for Context.join_nccl."""
    buf = C.create_string_buffer(128)
    check(lib().sgml_nccl_unique_id(buf))
    return buf.raw


def slab_plan(n: int, nranks: int, rank: int, replicate_n: int = 0) -> tuple[int, int, int]:
    """(vrep, z0, nz): levels < vrep are z-slabs; `rank` owns level-0 planes
    [z0, z0 + nz) of the 2^n + 1 (host only).  replicate_n as in
    SolverOptions (0: levels of <= 65 nodes per axis are replicated)."""
    v, z0, nz = C.c_int(), C.c_int(), C.c_int()
    check(lib().sgml_slab_plan_ex(n, nranks, rank, int(replicate_n), C.byref(v), C.byref(z0), C.byref(nz)))
    return v.value, z0.value, nz.value


_default_ctx: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


# --------------------------------------------------------------- field ----

class Field:
    """Device-resident fp64 field (grid.hpp:78-119), x-fastest order."""

    def __init__(self, grid: Grid, fill: float = 0.0, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.grid = grid
        self._h = C.c_void_p()
        check(lib().sgml_field_create(self.ctx.handle, grid.dim, grid.n, C.byref(self._h)))
        if fill != 0.0:
            self.fill(fill)

    @classmethod
    def from_numpy(cls, grid: Grid, values, ctx: Optional[Context] = None) -> "Field":
        f = cls(grid, ctx=ctx)
        f.upload(values)
        return f

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        return self.grid.total

    def upload(self, values) -> None:
        a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        if a.size != self.grid.total:
            raise ValueError("field upload: size mismatch")
        check(lib().sgml_field_upload(self._h, a.ctypes.data_as(_capi._D)))

    def numpy(self) -> np.ndarray:
        out = np.empty(self.grid.total, np.float64)
        check(lib().sgml_field_download(self._h, out.ctypes.data_as(_capi._D)))
        return out

    def fill(self, value: float) -> None:
        check(lib().sgml_field_fill(self._h, float(value)))

    def copy(self) -> "Field":
        f = Field(self.grid, ctx=self.ctx)
        check(lib().sgml_field_copy(f._h, self._h))
        return f

    def copy_from(self, other: "Field") -> None:
        check(lib().sgml_field_copy(self._h, other._h))

    def __del__(self):
        try:
            if self._h:
                lib().sgml_field_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def _h(f: Optional[Field]):
    return None if f is None else f.handle


class SolveState:
    """kernels.hpp:49-72: u/u_prev and du/du_prev double buffers."""

    def __init__(self, grid: Grid, ctx: Optional[Context] = None):
        self.u = Field(grid, ctx=ctx)
        self.u_prev = Field(grid, ctx=ctx)
        self.du = Field(grid, ctx=ctx)
        self.du_prev = Field(grid, ctx=ctx)
        self.level = 0

    def swap_buffers(self) -> None:
        self.u, self.u_prev = self.u_prev, self.u
        self.du, self.du_prev = self.du_prev, self.du

    def reset_level(self, v: int) -> None:
        self.level = v
        self.du.fill(0.0)
        self.du_prev.fill(0.0)


@dataclass
class OperatorCoefficients:
    """stencil.hpp:71-74"""
    sigma: Optional[Field] = None
    a: float = 0.0


# ------------------------------------------------------------- kernels ----

class _Work:
    """Optional accumulator standing in for the reference's ``std::uint64_t* work``."""

    def __init__(self, value: int = 0):
        self.value = value


def restriction_into(f: Field, v: int, bc: BoundarySpec, out: Field, scratch: Field,
                     work: Optional[_Work] = None) -> None:
    """kernels.cpp:305-325"""
    w = C.c_uint64(work.value if work else 0)
    check(lib().sgml_restriction_into(f.handle, v, C.byref(bc.to_c()), out.handle, scratch.handle,
                                      C.byref(w)))
    if work is not None:
        work.value = w.value


def restriction(f: Field, v: int, bc: BoundarySpec, work: Optional[_Work] = None) -> Field:
    """kernels.cpp:327-332"""
    out = Field(f.grid, ctx=f.ctx)
    scratch = Field(f.grid, ctx=f.ctx)
    restriction_into(f, v, bc, out, scratch, work)
    return out


def relaxation_interpolation(state: SolveState, g: Field, sigma_level: Optional[Field], a: float,
                             safety: float, bc: BoundarySpec, homogeneous: bool,
                             work: Optional[_Work] = None) -> float:
    """kernels.cpp:334-349: one pass at state.level; returns the unnormalised diag max."""
    d = C.c_double(0.0)
    w = C.c_uint64(work.value if work else 0)
    check(lib().sgml_relaxation_interpolation(
        state.u.handle, state.u_prev.handle, state.du.handle, state.du_prev.handle, state.level,
        g.handle, _h(sigma_level), float(a), float(safety), C.byref(bc.to_c()), int(bool(homogeneous)),
        C.byref(d), C.byref(w)))
    if work is not None:
        work.value = w.value
    return d.value


def residual_update(r: Field, e: Field, coeff: OperatorCoefficients, bc: BoundarySpec) -> None:
    """kernels.cpp:351-358"""
    check(lib().sgml_residual_update(r.handle, e.handle, _h(coeff.sigma), float(coeff.a),
                                     C.byref(bc.to_c())))


def residual(u: Field, f: Field, coeff: OperatorCoefficients, bc: BoundarySpec) -> Field:
    """kernels.cpp:360-365"""
    r = f.copy()
    residual_update(r, u, coeff, bc)
    return r


def max_abs(f: Field) -> float:
    out = C.c_double(0.0)
    check(lib().sgml_max_abs(f.handle, C.byref(out)))
    return out.value


def trapezoid_mean(f: Field) -> float:
    out = C.c_double(0.0)
    check(lib().sgml_trapezoid_mean(f.handle, C.byref(out)))
    return out.value


def zero_mean_projection(f: Field) -> None:
    check(lib().sgml_zero_mean_projection(f.handle))


def apply_boundary(u: Field, bc: BoundarySpec, homogeneous: bool) -> None:
    check(lib().sgml_apply_boundary(u.handle, C.byref(bc.to_c()), int(bool(homogeneous))))


def pure_neumann_pin(u: Field) -> None:
    """cycle.cpp:135-138"""
    check(lib().sgml_pure_neumann_pin(u.handle))


def restrict_sigma_levels(sigma: Field, n: int) -> list:
    """cycle.cpp:117-133 (empty list for an absent coefficient)."""
    if sigma is None:
        return []
    levels = [Field(sigma.grid, ctx=sigma.ctx) for _ in range(n)]
    arr = (C.c_void_p * n)(*[lv.handle.value for lv in levels])
    check(lib().sgml_restrict_sigma_levels(sigma.handle, arr))
    return levels


# ------------------------------------------------------------ schedule ----

@dataclass
class ScheduleStep:
    """cycle.hpp:33-38"""
    RESTRICT_SOURCE = 0
    RELAX = 1
    kind: int = 1
    level: int = 0
    count: int = 1


@dataclass
class CycleSchedule:
    n: int = 0
    n_r: int = 1
    steps: list = field(default_factory=list)


def build_schedule(n: int, n_r: int) -> CycleSchedule:
    """cycle.cpp:28-45 (ValueError for n < 1 or n_r < 1)."""
    cap = 8192
    k, lv, cn = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
    count = C.c_int(0)
    check(lib().sgml_build_schedule(n, n_r, k, lv, cn, cap, C.byref(count)))
    return CycleSchedule(n, n_r, [ScheduleStep(k[i], lv[i], cn[i]) for i in range(count.value)])


def closed_form_work_units(n: int, n_r: int) -> int:
    return int(lib().sgml_closed_form_work_units(n, n_r))


def schedule_work_units(schedule: CycleSchedule) -> int:
    return sum(st.level if st.kind == ScheduleStep.RESTRICT_SOURCE else st.count
               for st in schedule.steps)


# -------------------------------------------------------------- driver ----

@dataclass
class SolverConfig:
    """cycle.hpp:66-71"""
    n_r: int = 2
    tol: float = 1e-12
    max_cycles: int = 50
    safety: float = 0.9

    def to_c(self) -> _capi.SolverCfg:
        return _capi.SolverCfg(self.n_r, self.max_cycles, self.tol, self.safety)


@dataclass
class SolverOptions:
    """Engine switches with no reference counterpart."""
    engine: str = "compact"     # "compact" (B200 level-compact) or "literal" (reference-shaped)
    use_graph: bool = True      # replay each cycle from a CUDA graph (single-GPU compact solves)
    timing: bool = False
    timing_classes: int = 0     # 0: time every kernel class; else a mask of 1 << class index
    stencil: str = "radial"     # "radial" (the reference's) or "compact" 5/7-point (no reference)
    small_levels: bool = True   # one CTA per visit of a small level array (else one launch per pass)
    cluster_levels: bool = True  # small-level operations batched into cluster launches (single GPU)
    replicate_n: int = 0        # z-slab solves: replicate levels of <= this many nodes per axis (0: 65)

    def to_c(self) -> _capi.SolverOpts:
        if self.stencil not in ("radial", "compact"):
            raise ValueError("stencil must be 'radial' or 'compact'")
        return _capi.SolverOpts(0 if self.engine == "compact" else 1, 1 if self.use_graph else -1,
                                int(self.timing), int(self.timing_classes),
                                0 if self.stencil == "radial" else 1, 0 if self.small_levels else -1,
                                0 if self.cluster_levels else -1, int(self.replicate_n))


@dataclass
class DiagSample:
    cycle: int
    pass_: int
    level: int
    value: float


@dataclass
class CycleRecord:
    cycle: int
    work_units: int
    residual: float
    diag_min: float
    l1_error: Optional[float] = None


@dataclass
class SolveReport:
    rows: list = field(default_factory=list)
    trace: list = field(default_factory=list)
    converged: bool = False
    nan_detected: bool = False
    stagnated: bool = False
    normalization: float = 0.0
    node_updates: int = 0
    device_ms: float = 0.0
    kernel_launches: int = 0


ExactSolution = Callable[[np.ndarray, np.ndarray, np.ndarray], np.ndarray]


@dataclass
class ProblemSpec:
    """cycle.hpp:106-115 with host numpy fields (f, sigma) of grid.total values."""
    grid: Grid
    f: np.ndarray
    bc: BoundarySpec = field(default_factory=BoundarySpec)
    sigma: Optional[np.ndarray] = None
    a: float = 0.0
    exact: Optional[ExactSolution] = None


@dataclass
class SolveResult:
    u: np.ndarray
    report: SolveReport


class _ReportBuffers:
    def __init__(self, rows_cap: int = 4096, trace_cap: int = 1 << 16):
        self.rows = (_capi.CycleRecord * rows_cap)()
        self.trace = (_capi.DiagSample * trace_cap)()
        self.c = _capi.Report()
        self.c.rows, self.c.rows_cap = C.cast(self.rows, C.POINTER(_capi.CycleRecord)), rows_cap
        self.c.trace, self.c.trace_cap = C.cast(self.trace, C.POINTER(_capi.DiagSample)), trace_cap

    def to_report(self) -> SolveReport:
        c = self.c
        rep = SolveReport()
        for i in range(min(c.n_rows, c.rows_cap)):
            r = self.rows[i]
            rep.rows.append(CycleRecord(r.cycle, int(r.work_units), r.residual, r.diag_min,
                                        r.l1_error if r.has_l1 else None))
        for i in range(min(c.n_trace, c.trace_cap)):
            t = self.trace[i]
            rep.trace.append(DiagSample(t.cycle, t.pass_, t.level, t.value))
        rep.converged, rep.nan_detected, rep.stagnated = bool(c.converged), bool(c.nan_detected), \
            bool(c.stagnated)
        rep.normalization, rep.node_updates = c.normalization, int(c.node_updates)
        rep.device_ms, rep.kernel_launches = c.device_ms, int(c.kernel_launches)
        return rep


def _l1_hook(grid: Grid, exact: ExactSolution):
    """problems.cpp:195-215 (l1 against the exact solution), evaluated on the host."""
    N = grid.N
    idx = np.arange(N, dtype=np.float64) * grid.h
    axes = np.meshgrid(*([idx] * grid.dim), indexing="ij")[::-1] if grid.dim == 2 else None
    if grid.dim == 2:
        y, x = np.meshgrid(idx, idx, indexing="ij")
        z = np.zeros_like(x)
    else:
        z, y, x = np.meshgrid(idx, idx, idx, indexing="ij")
    del axes
    ue = np.asarray(exact(x, y, z), np.float64).reshape(-1)
    w1 = np.ones(N)
    w1[0] = w1[-1] = 0.5
    w = w1
    for _ in range(grid.dim - 1):
        w = np.multiply.outer(w1, w)
    w = w.reshape(-1)
    den = float(np.sum(w * np.abs(ue)))

    def hook(_user, _cycle, field_ptr, out):
        n = grid.total
        buf = np.empty(n, np.float64)
        rc = lib().sgml_field_download(field_ptr, buf.ctypes.data_as(_capi._D))
        if rc != 0 or den == 0.0:
            return 0
        out[0] = float(np.sum(w * np.abs(buf - ue))) / den
        return 1

    return _capi.HOOK(hook)


def solve(problem: ProblemSpec, config: SolverConfig = SolverConfig(),
          options: Optional[SolverOptions] = None, ctx: Optional[Context] = None) -> SolveResult:
    """cycle.cpp:140-247, end to end through ``sgml_solve`` (host f in, host u out)."""
    ctx = ctx or default_context()
    g = problem.grid
    f = np.ascontiguousarray(problem.f, np.float64).reshape(-1)
    if f.size != g.total:
        raise ValueError("solve: source grid mismatch")
    sig = None
    if problem.sigma is not None:
        sig = np.ascontiguousarray(problem.sigma, np.float64).reshape(-1)
        if sig.size != g.total:
            raise ValueError("solve: sigma grid mismatch")
    u = np.empty(g.total, np.float64)
    rb = _ReportBuffers()
    hook = None
    if problem.exact is not None:
        hook = _l1_hook(g, problem.exact)
        rb.c.hook = hook
    opts = (options or SolverOptions()).to_c()
    check(lib().sgml_solve(ctx.handle, g.dim, g.n, C.byref(problem.bc.to_c()),
                           f.ctypes.data_as(_capi._D),
                           None if sig is None else sig.ctypes.data_as(_capi._D), float(problem.a),
                           C.byref(config.to_c()), C.byref(opts), u.ctypes.data_as(_capi._D),
                           C.byref(rb.c)))
    return SolveResult(u, rb.to_report())


def solve_many(problems: Sequence[ProblemSpec], config: SolverConfig = SolverConfig(),
               options: Optional[SolverOptions] = None, ctx: Optional[Context] = None,
               out: Optional[Sequence[np.ndarray]] = None) -> list:
    """Several solves of one problem shape (same grid, bc, a, sigma; different
    sources) through ``sgml_solve_many``: transfers of neighbouring solves
    overlap the device work.  Same results as one ``solve`` per problem.
    ``out``: optional host arrays (pinned for full overlap) for the solutions."""
    ctx = ctx or default_context()
    if not problems:
        return []
    p0 = problems[0]
    g = p0.grid
    fs = [np.ascontiguousarray(p.f, np.float64).reshape(-1) for p in problems]
    bc0 = bytes(p0.bc.to_c())
    sig = None
    if p0.sigma is not None:
        sig = np.ascontiguousarray(p0.sigma, np.float64).reshape(-1)
    for p, f in zip(problems, fs):
        if p.grid != g or f.size != g.total:
            raise ValueError("solve_many: every problem must share the grid")
        if bytes(p.bc.to_c()) != bc0 or float(p.a) != float(p0.a):
            raise ValueError("solve_many: every problem must share bc and a")
        if (p.sigma is None) != (sig is None) or (
                sig is not None and p.sigma is not p0.sigma
                and not np.array_equal(np.asarray(p.sigma, np.float64).reshape(-1), sig)):
            raise ValueError("solve_many: every problem must share sigma")
        if p.exact is not None:
            raise ValueError("solve_many: exact solutions (l1 rows) need solve()")
    if out is not None:
        if len(out) != len(problems):
            raise ValueError("solve_many: one output array per problem")
        for u in out:
            if not (isinstance(u, np.ndarray) and u.dtype == np.float64 and u.flags.c_contiguous
                    and u.size == g.total):
                raise ValueError("solve_many: outputs must be C-contiguous float64 arrays of grid.total")
    us = list(out) if out is not None else [np.empty(g.total, np.float64) for _ in problems]
    rbs = [_ReportBuffers() for _ in problems]
    reps = (_capi.Report * len(problems))(*[rb.c for rb in rbs])
    fptr = (_capi._D * len(problems))(*[f.ctypes.data_as(_capi._D) for f in fs])
    uptr = (_capi._D * len(problems))(*[u.ctypes.data_as(_capi._D) for u in us])
    opts = (options or SolverOptions()).to_c()
    check(lib().sgml_solve_many(ctx.handle, g.dim, g.n, C.byref(p0.bc.to_c()), len(problems), fptr,
                                None if sig is None else sig.ctypes.data_as(_capi._D), float(p0.a),
                                C.byref(config.to_c()), C.byref(opts), uptr, reps))
    for rb, rc in zip(rbs, reps):
        rb.c = rc
    return [SolveResult(u, rb.to_report()) for u, rb in zip(us, rbs)]


class Solver:
    """Preallocated device engine for repeated solves of one problem shape."""

    def __init__(self, grid: Grid, bc: BoundarySpec, a: float = 0.0, sigma: Optional[Field] = None,
                 config: SolverConfig = SolverConfig(), options: Optional[SolverOptions] = None,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.grid = grid
        self._h = C.c_void_p()
        check(lib().sgml_solver_create(self.ctx.handle, grid.dim, grid.n, C.byref(bc.to_c()),
                                       float(a), _h(sigma), C.byref(config.to_c()),
                                       C.byref((options or SolverOptions()).to_c()),
                                       C.byref(self._h)))
        self._rb = _ReportBuffers()

    def run(self, f: Field, u_out: Optional[Field] = None) -> SolveReport:
        self._rb.c.n_rows = self._rb.c.n_trace = 0
        check(lib().sgml_solver_run(self._h, f.handle, _h(u_out), C.byref(self._rb.c)))
        return self._rb.to_report()

    def footprint(self) -> int:
        b = C.c_uint64(0)
        check(lib().sgml_solver_footprint(self._h, C.byref(b)))
        return b.value

    def __del__(self):
        try:
            if self._h:
                lib().sgml_solver_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def single_cycle(state: SolveState, source: Field, sigma_levels: Sequence[Field], a: float,
                 bc: BoundarySpec, homogeneous: bool, schedule: CycleSchedule, safety: float,
                 cycle_index: int, normalization: float, report: SolveReport, work: _Work,
                 options: Optional[SolverOptions] = None) -> None:
    """cycle.cpp:76-111: one cycle; the correction lands in state.u."""
    rb = _ReportBuffers(rows_cap=1)
    n = source.grid.n
    levels = None
    if sigma_levels:
        levels = (C.c_void_p * n)(*[lv.handle.value for lv in sigma_levels])
    w = C.c_uint64(work.value)
    opts = (options or SolverOptions()).to_c()
    try:
        check(lib().sgml_single_cycle(source.ctx.handle, state.u.handle, source.handle, levels,
                                      float(a), C.byref(bc.to_c()), int(bool(homogeneous)),
                                      schedule.n_r, float(safety), int(cycle_index),
                                      float(normalization), C.byref(opts), C.byref(rb.c), C.byref(w)))
    finally:
        work.value = w.value
        report.trace.extend(rb.to_report().trace)


def single_cycle_state(state: SolveState, source: Field, sigma_levels: Sequence[Field], a: float,
                       bc: BoundarySpec, homogeneous: bool, schedule: CycleSchedule, safety: float,
                       cycle_index: int, normalization: float, report: SolveReport, work: _Work) -> None:
    """cycle.cpp:76-111 with the reference's full SolveState semantics (the C++
    drop-in's single_cycle): the cycle starts from state.u, runs the
    schedule's own steps with the given sigma levels (one per level, or none),
    and leaves u, u_prev, du, du_prev and level as the reference does, also
    when a pass raises kernel_error (the literal kernels, pass by pass)."""
    n = len(schedule.steps)
    kinds = (C.c_int * max(n, 1))(*[int(st.kind) for st in schedule.steps])
    levels = (C.c_int * max(n, 1))(*[int(st.level) for st in schedule.steps])
    counts = (C.c_int * max(n, 1))(*[int(st.count) for st in schedule.steps])
    passes = sum(int(st.count) for st in schedule.steps if int(st.kind) == 1)
    rb = _ReportBuffers(rows_cap=1, trace_cap=max(passes, 1))
    lv = None
    if sigma_levels:
        lv = (C.c_void_p * len(sigma_levels))(*[f.handle.value for f in sigma_levels])
    level = C.c_int(state.level)
    w = C.c_uint64(work.value)
    try:
        check(lib().sgml_single_cycle_state(source.ctx.handle, state.u.handle, state.u_prev.handle, state.du.handle,
                                            state.du_prev.handle, C.byref(level), source.handle, lv, float(a),
                                            C.byref(bc.to_c()), int(bool(homogeneous)), kinds, levels, counts, n,
                                            float(safety), int(cycle_index), float(normalization), C.byref(rb.c),
                                            C.byref(w)))
    finally:
        work.value = w.value
        state.level = level.value
        report.trace.extend(rb.to_report().trace)


Work = _Work
