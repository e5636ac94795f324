"""Post-solve fields of the reference's experiments (problems.hpp:100-148)
on the device: difference fields, deformation velocity, node motion and RK4
streamlines.  Each call runs the sm_100a kernels of csrc/fields.cu through
the C-ABI; results are the reference's bits (problems.cpp:40-97, 327-455).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import check, lib
from .api import Field, Grid

__all__ = ["VectorField", "StreamlineStop", "Streamline", "axis_derivative", "gradient", "curl", "divergence",
           "deformation_velocity", "move_nodes", "sample_vector", "integrate_streamline",
           "integrate_streamlines", "poisson2d_source", "poisson3d_source", "sinsin2d_source",
           "capacitor_sigma", "trifoil_sources", "deformation_sources", "write_field_vtk", "write_vector_vtk"]


def _handles(fields: Sequence[Optional[Field]]):
    arr = (C.c_void_p * len(fields))(*[f.handle.value if f is not None else None for f in fields])
    return arr


class VectorField:
    """problems.hpp:31-39: three component fields, comp[2] unused in 2D."""

    def __init__(self, grid: Grid, comps: Optional[Sequence[Field]] = None, ctx=None):
        self.grid = grid
        self.dim = grid.dim
        if comps is None:
            comps = [Field(grid, ctx=ctx) for _ in range(3)]
        self.comp = list(comps)

    @classmethod
    def from_numpy(cls, grid: Grid, arrays, ctx=None) -> "VectorField":
        comps = [Field.from_numpy(grid, a, ctx=ctx) for a in arrays]
        while len(comps) < 3:
            comps.append(Field(grid, ctx=ctx))
        return cls(grid, comps)

    def numpy(self) -> np.ndarray:
        return np.stack([c.numpy() for c in self.comp])


class StreamlineStop(enum.IntEnum):
    """problems.hpp:139"""
    max_steps = 0
    left_domain = 1
    stagnation = 2


@dataclass
class Streamline:
    points: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    stop: StreamlineStop = StreamlineStop.max_steps


def axis_derivative(u: Field, axis: int) -> Field:
    """problems.cpp:74-97"""
    out = Field(u.grid, ctx=u.ctx)
    check(lib().sgml_axis_derivative(u.handle, int(axis), out.handle))
    return out


def gradient(u: Field) -> VectorField:
    """problems.cpp:391-396"""
    v = VectorField(u.grid, ctx=u.ctx)
    check(lib().sgml_gradient(u.handle, _handles(v.comp)))
    return v


def curl(psi: VectorField) -> VectorField:
    """problems.cpp:376-389 (3D only: ValueError otherwise)"""
    v = VectorField(psi.grid, ctx=psi.comp[0].ctx)
    check(lib().sgml_curl(_handles(psi.comp), _handles(v.comp)))
    return v


def divergence(v: VectorField) -> Field:
    """problems.cpp:398-405"""
    out = Field(v.grid, ctx=v.comp[0].ctx)
    check(lib().sgml_divergence(_handles(v.comp), out.handle))
    return out


def deformation_velocity(u: Field, f_raw: Field, raw_integral: float, t: float) -> VectorField:
    """problems.cpp:327-341 (ValueError on a zero denominator)"""
    v = VectorField(u.grid, ctx=u.ctx)
    check(lib().sgml_deformation_velocity(u.handle, f_raw.handle, float(raw_integral), float(t),
                                          _handles(v.comp)))
    return v


def move_nodes(u: Field, f_raw: Field, raw_integral: float, t: float, steps: int) -> VectorField:
    """problems.cpp:343-372: node positions as coordinate fields (x, y, z)."""
    pos = VectorField(u.grid, ctx=u.ctx)
    check(lib().sgml_move_nodes(u.handle, f_raw.handle, float(raw_integral), float(t), int(steps),
                                _handles(pos.comp)))
    return pos


def sample_vector(v: VectorField, points) -> np.ndarray:
    """problems.cpp:407-413 at one point (3,) or many (m, 3)."""
    p = np.ascontiguousarray(points, np.float64)
    one = p.ndim == 1
    p = p.reshape(-1, 3)
    out = np.zeros_like(p)
    check(lib().sgml_sample_vector(_handles(v.comp), v.dim, p.ctypes.data_as(_capi._D), p.shape[0],
                                   out.ctypes.data_as(_capi._D)))
    return out[0] if one else out


def integrate_streamlines(v: VectorField, seeds, step: float, max_steps: int) -> list:
    """problems.cpp:415-455 for several seeds (one device thread each)."""
    sd = np.ascontiguousarray(seeds, np.float64).reshape(-1, 3)
    m = sd.shape[0]
    pts = np.zeros((m, max_steps + 1, 3))
    counts = np.zeros(m, np.int32)
    stops = np.zeros(m, np.int32)
    check(lib().sgml_integrate_streamlines(_handles(v.comp), sd.ctypes.data_as(_capi._D), m, float(step),
                                           int(max_steps), pts.ctypes.data_as(_capi._D),
                                           counts.ctypes.data_as(C.POINTER(C.c_int)),
                                           stops.ctypes.data_as(C.POINTER(C.c_int))))
    return [Streamline(pts[s, :counts[s]].copy(), StreamlineStop(int(stops[s]))) for s in range(m)]


def integrate_streamline(v: VectorField, seed, step: float, max_steps: int) -> Streamline:
    """problems.cpp:415-455"""
    return integrate_streamlines(v, [seed], step, max_steps)[0]


# ---- problem builders on the device -------------------
# The reference's sources / coefficients (problems.cpp) as device fields, bit
# for bit: libm runs on the host over the few distinct arguments, the device
# assembles the dense field.

def poisson2d_source(grid: Grid, ctx=None) -> Field:
    """problems.cpp:160-176"""
    f = Field(grid, ctx=ctx)
    check(lib().sgml_build_poisson2d_source(f.handle))
    return f


def poisson3d_source(grid: Grid, ctx=None) -> Field:
    """problems.cpp:178-193"""
    f = Field(grid, ctx=ctx)
    check(lib().sgml_build_poisson3d_source(f.handle))
    return f


def sinsin2d_source(grid: Grid, ctx=None) -> Field:
    """BASELINE.json configs[0]: f = -2 pi^2 sin(pi x) sin(pi y)"""
    f = Field(grid, ctx=ctx)
    check(lib().sgml_build_sinsin2d_source(f.handle))
    return f


def capacitor_sigma(grid: Grid, mode: str = "high", ctx=None) -> Field:
    """problems.cpp:500-521 ("high": strongly conducting sphere, "low": weakly)"""
    if mode not in ("high", "low"):
        raise ValueError('capacitor_problem: mode must be "high" or "low"')
    s = Field(grid, ctx=ctx)
    check(lib().sgml_build_capacitor_sigma(s.handle, 1 if mode == "high" else 0))
    return s


def trifoil_sources(grid: Grid, r: float = 0.14, ctx=None) -> list:
    """problems.cpp:374-398: the sources -omega_c of the three psi problems."""
    fs = [Field(grid, ctx=ctx) for _ in range(3)]
    check(lib().sgml_build_trifoil_sources(_handles(fs), float(r)))
    return fs


def deformation_sources(points, grid: Grid, ctx=None):
    """problems.cpp:302-325 for a closed curve: (f, f_raw, raw_integral)."""
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    f, f_raw = Field(grid, ctx=ctx), Field(grid, ctx=ctx)
    ri = C.c_double(0.0)
    check(lib().sgml_build_deformation_sources(pts.ctypes.data_as(_capi._D), pts.shape[0], f.handle, f_raw.handle,
                                               C.byref(ri)))
    return f, f_raw, ri.value


# ---- output (io.cpp:14-64): streamed from the device ------------------------

def write_field_vtk(f: Field, path: str, name: str) -> None:
    """io.cpp:45-53, byte for byte."""
    check(lib().sgml_write_field_vtk(f.handle, str(path).encode(), name.encode()))


def write_vector_vtk(v: VectorField, path: str, name: str) -> None:
    """io.cpp:55-64, byte for byte (the third component of a 2D field is written as 0)."""
    comps = list(v.comp[:3]) if v.dim == 3 else [v.comp[0], v.comp[1], None]
    check(lib().sgml_write_vector_vtk(_handles(comps), str(path).encode(), name.encode()))
