"""Shared deterministic test cases (boundary sets, LCG inputs, problems).

Used by the golden-vector generator (tests/golden/make_golden.py), the CPU
oracle tests and the GPU parity tests so all three see identical inputs.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (test infrastructure)

D, NEU = O.DIRICHLET, O.NEUMANN

# name -> (kinds[6], values[6])
BCS = {
    "dir0": ([D] * 6, [0.0] * 6),
    "dir_quarter": ([D] * 6, [0.25] * 6),
    "neumann": ([NEU] * 6, [0.0] * 6),
    # capacitor-like: z plates Dirichlet -1/+1, lateral Neumann (problems.cpp:517-519)
    "plates": ([NEU, NEU, NEU, NEU, D, D], [0, 0, 0, 0, -1.0, 1.0]),
    # 2D mixed: x faces Dirichlet (distinct values: corner tie-break), y faces Neumann
    "mixed_x": ([D, D, NEU, NEU, NEU, NEU], [0.5, -0.75, 0, 0, 0, 0]),
    # every face Dirichlet with distinct values (lowest face id wins at edges)
    "dir_distinct": ([D] * 6, [1.0, -2.0, 3.0, -4.0, 5.0, -6.0]),
    # high faces Neumann, low faces Dirichlet (exercises the F5 wrap reads)
    "low_dir_high_neu": ([D, NEU, D, NEU, D, NEU], [0.3, 0, -0.2, 0, 0.1, 0]),
    # x faces Dirichlet (distinct values), every other face Neumann: the
    # x-high face column next to Neumann rows / planes (corner mirror ghosts)
    "xdir_yzneu": ([D, D, NEU, NEU, NEU, NEU], [0.5, -0.75, 0, 0, 0, 0]),
}


def bc(name: str) -> O.Bc:
    k, v = BCS[name]
    return O.make_bc(k, v)


def sigma_field(g, seed: int) -> np.ndarray:
    """Positive heterogeneous coefficient in [0.6, 1.4] (kernels_tests.cpp:249-255 style)."""
    return 1.0 + 0.4 * O.lcg(g, seed)


def canon(a: np.ndarray) -> np.ndarray:
    """Bit pattern with -0.0 canonicalised to +0.0."""
    a = np.asarray(a, np.float64).copy()
    a[a == 0.0] = 0.0
    return a.view(np.uint64)


def bits_equal(a, b) -> bool:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return bool(np.array_equal(canon(np.where(na, 0, a)), canon(np.where(nb, 0, b))))


# kernel-level relax cases: (dim, n, level, bc, with_sigma, a, homogeneous)
def relax_cases(full: bool = True):
    out = []
    for dim, n in ((2, 4), (3, 3)) + (((2, 5), (3, 4)) if full else ()):
        for level in range(0, n):
            for bcn in ("dir0", "neumann", "plates" if dim == 3 else "mixed_x", "dir_distinct",
                        "low_dir_high_neu"):
                for sig in (False, True):
                    for a, hom in ((0.0, False), (0.7, True), (-0.3, False)):
                        out.append((dim, n, level, bcn, sig, a, hom))
    return out


def relax_inputs(dim, n, level, bcn, sig, a, hom):
    g = O.make_grid(dim, n)
    seed = 1000 * dim + 100 * n + 10 * level + (7 if sig else 0)
    up = O.lcg(g, seed + 3)
    dup = O.lcg(g, seed + 5)
    gs = O.lcg(g, seed + 9)
    s = sigma_field(g, seed + 13) if sig else None
    return g, bc(bcn), up, dup, gs, s


def poisson_sinsin_2d(g) -> np.ndarray:
    return O.fill("sinsin2d", g)


# solve cases: name -> builder returning (grid, bc, f, sigma, a)
def solve_problem(name: str, n: int):
    if name == "sinsin2d":
        g = O.make_grid(2, n)
        return g, bc("dir0"), O.fill("sinsin2d", g), None, 0.0
    if name == "poisson2d":
        g = O.make_grid(2, n)
        return g, bc("dir0"), O.fill("poisson2d", g), None, 0.0
    if name == "poisson3d":
        g = O.make_grid(3, n)
        return g, bc("dir0"), O.fill("poisson3d", g), None, 0.0
    if name in ("capacitor_high", "capacitor_low"):
        g = O.make_grid(3, n)
        sig = O.fill("capacitor_sigma", g, -1.0 if name.endswith("high") else 1.0)
        return g, bc("plates"), np.zeros(g.total), sig, 0.0
    if name == "neumann2d_a":
        # all-Neumann, a = 0.1, compatible cosine source (cycle_tests.cpp:150-177 shape)
        g = O.make_grid(2, n)
        x = np.arange(g.N) * g.h
        yy, xx = np.meshgrid(x, x, indexing="ij")
        f = (-2.0 * math.pi ** 2 * np.cos(math.pi * xx) * np.cos(math.pi * yy)).reshape(-1)
        return g, bc("neumann"), f, None, 0.1
    if name == "neumann2d":
        g = O.make_grid(2, n)
        x = np.arange(g.N) * g.h
        yy, xx = np.meshgrid(x, x, indexing="ij")
        f = (-2.0 * math.pi ** 2 * np.cos(math.pi * xx) * np.cos(math.pi * yy)).reshape(-1)
        return g, bc("neumann"), f, None, 0.0
    if name == "mixed2d":
        g = O.make_grid(2, n)
        return g, bc("mixed_x"), O.fill("sinsin2d", g), None, 0.0
    if name == "mixed3d_a":
        g = O.make_grid(3, n)
        return g, bc("low_dir_high_neu"), O.fill("poisson3d", g), None, -0.3
    if name == "neumann3d_a":
        # all-Neumann 3D, a = 0.1, compatible cosine source
        g = O.make_grid(3, n)
        x = np.arange(g.N) * g.h
        zz, yy, xx = np.meshgrid(x, x, x, indexing="ij")
        f = (-3.0 * math.pi ** 2 * np.cos(math.pi * xx) * np.cos(math.pi * yy) * np.cos(math.pi * zz)).reshape(-1)
        return g, bc("neumann"), f, None, 0.1
    if name == "sigma3d_dirichlet":
        g = O.make_grid(3, n)
        return g, bc("dir_distinct"), O.fill("poisson3d", g), sigma_field(g, 77), 0.0
    if name == "sigma2d_mixed_a":
        # 2D: sigma + x faces Dirichlet (distinct values) / y faces Neumann + a
        g = O.make_grid(2, n)
        return g, bc("mixed_x"), O.fill("sinsin2d", g), sigma_field(g, 91), 0.2
    if name == "sigma2d_neumann_a":
        # 2D all-Neumann with sigma and a = 0.1 (cosine source)
        g = O.make_grid(2, n)
        x = np.arange(g.N) * g.h
        yy, xx = np.meshgrid(x, x, indexing="ij")
        f = (-2.0 * math.pi ** 2 * np.cos(math.pi * xx) * np.cos(math.pi * yy)).reshape(-1)
        return g, bc("neumann"), f, sigma_field(g, 93), 0.1
    if name == "mixed2d_a":
        # 2D low faces Dirichlet / high faces Neumann (the F5 wrap reads), a = 0.15
        g = O.make_grid(2, n)
        return g, bc("low_dir_high_neu"), O.fill("sinsin2d", g), None, 0.15
    if name == "sigma3d_mixed_a":
        g = O.make_grid(3, n)
        return g, bc("low_dir_high_neu"), O.fill("poisson3d", g), sigma_field(g, 95), 0.2
    if name == "zero_source_dirichlet1":
        g = O.make_grid(2, n)
        return g, bc("dir_quarter"), np.zeros(g.total), None, 0.0
    raise KeyError(name)


SOLVE_CASES = [
    ("sinsin2d", 4), ("sinsin2d", 6), ("poisson2d", 5), ("poisson3d", 3), ("poisson3d", 4),
    ("capacitor_high", 3), ("capacitor_low", 4), ("neumann2d_a", 4), ("neumann2d", 5),
    ("mixed2d", 5), ("mixed3d_a", 3), ("sigma3d_dirichlet", 3), ("zero_source_dirichlet1", 3),
]

# Solves large enough that the level-0 (and coarser) arrays exceed the
# one-CTA small-level path (2D > 65^2, 3D > 17^3), so the TMA relaxation
# kernels run with sigma, a != 0, all-Neumann and mixed faces.
# Every relaxation-kernel specialisation at sizes where the TMA kernels carry
# the large levels (2D 129^2, 3D 33^3): (dim, n, bc, sigma, a)
SPEC_CASES = [(dim, n, bcn, sig, a)
              for dim, n in ((2, 7), (3, 5))
              for bcn in ("dir_distinct", "neumann", "xdir_yzneu", "low_dir_high_neu")
              for sig in (False, True) for a in (0.0, 0.25)]


def spec_key(dim, n, bcn, sig, a) -> str:
    return f"spec:{dim}:{n}:{bcn}:{int(sig)}:{a}"


def spec_problem(dim, n, bcn, sig, a):
    g = O.make_grid(dim, n)
    f = O.fill("sinsin2d" if dim == 2 else "poisson3d", g)
    return g, bc(bcn), f, (sigma_field(g, 57 + dim) if sig else None), a


SOLVE_CASES_LARGE = [
    ("sigma2d_mixed_a", 7), ("sigma2d_neumann_a", 7), ("neumann2d_a", 8), ("mixed2d_a", 8),
    ("sigma2d_mixed_a", 8), ("neumann3d_a", 5), ("sigma3d_mixed_a", 5), ("sigma3d_dirichlet", 5),
]


# ------------------------------------------------- post-solve fields ----
# problems.cpp:40-97, 327-455 on deterministic inputs (tests/golden, parity)

FIELD_GRIDS = [(2, 3), (2, 5), (3, 3), (3, 4)]


def field_inputs(dim: int, n: int) -> dict:
    g = O.make_grid(dim, n)
    T = g.total
    u = O.lcg(g, 101 + dim)
    psi = np.stack([O.lcg(g, 111 + c) for c in range(3)])
    v = np.stack([O.lcg(g, 121 + c) for c in range(dim)])
    f_raw = np.abs(O.lcg(g, 131)) + 0.25
    # a smooth swirl (streamlines that run for many steps) plus a random field
    x = (np.arange(T) % g.N) * g.h
    y = ((np.arange(T) // g.N) % g.N) * g.h
    swirl = [-(y - 0.5), x - 0.5] + ([0.1 * np.ones(T)] if dim == 3 else [])
    seeds = np.array([[0.7, 0.5, 0.5], [0.31, 0.62, 0.44], [0.5, 0.5, 0.5], [1.2, 0.5, 0.5]])
    if dim == 2:
        seeds[:, 2] = 0.0
    return {"g": g, "u": u, "psi": psi, "v": v, "f_raw": f_raw, "swirl": np.stack(swirl),
            "seeds": seeds, "raw_integral": 1.5, "t": 0.35, "steps": 6, "step": 0.02, "max_steps": 120}
