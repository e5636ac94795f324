"""Reference parity at the BASELINE.json configuration sizes.

tests/golden/large.json holds what the UNMODIFIED reference solver computed
for each case (tests/golden/make_golden_large.py, run once where
/root/reference exists): the residual history (hex of every CycleRecord),
flags, normalisation, node updates, trace digest and the sha256 of the
canonical solution bits.  Here the B200 engine solves the same problems,
its inputs built ON THE DEVICE by the repo's builders (their digest must
equal the reference builders' first), and everything is compared bit for
bit:

  capacitor high / low at 129^3 and 257^3  (problems.cpp:500-521, sigma,
                                           lateral Neumann, f = 0)
  trifoil psi_x / psi_y / psi_z at 513^3   (problems.cpp:378-410, r = 0.14)
  deformation 2049^2                       (problems.cpp:302-325, all-Neumann,
                                           a = 0.1, CLI smoke circle)
  deformation 2049^2, mixed faces          (x / y
                                           component of the vector Laplace)
  Poisson 513^3                            (problems.cpp:178-193, the bench)
"""
import functools
import hashlib
import json
import math
import os

import numpy as np
import pytest

import cases as K
import paper_1703_07206_b200 as S

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
LARGE_JSON = os.path.join(HERE, "golden", "large.json")
CASES = ["capacitor_high@7", "capacitor_low@7", "capacitor_high@8", "capacitor_low@8",
         "deformation_circle@11", "deformation_mixed_x@11", "deformation_mixed_y@11",
         "trifoil_x@9", "trifoil_y@9", "trifoil_z@9", "poisson3d@9", "poisson3d@8"]
CFG = S.SolverConfig(n_r=2, tol=1e-10, max_cycles=60, safety=0.9)


@functools.lru_cache(maxsize=1)
def golden():
    return json.load(open(LARGE_JSON)) if os.path.exists(LARGE_JSON) else {}


def digest(a) -> str:
    return hashlib.sha256(K.canon(np.asarray(a, np.float64)).tobytes()).hexdigest()


def circle():
    # the CLI smoke circle (cli_smoke.cpp:121-130): 32 points, centre (1/2, 1/2), radius 1/4
    return [[0.5 + 0.25 * math.cos(2.0 * math.pi * q / 32.0), 0.5 + 0.25 * math.sin(2.0 * math.pi * q / 32.0), 0.0]
            for q in range(32)]


@functools.lru_cache(maxsize=2)
def trifoil(n):
    return S.trifoil_sources(S.make_grid(3, n), 0.14)


def problem(case):
    """(grid, bc, a, f Field, sigma Field | None), device-built."""
    name, n = case.rsplit("@", 1)
    n = int(n)
    D, N = S.BcKind.dirichlet, S.BcKind.neumann
    if name == "poisson3d":
        g = S.make_grid(3, n)
        return g, S.BoundarySpec.all_dirichlet(0.0), 0.0, S.poisson3d_source(g), None
    if name.startswith("capacitor_"):
        g = S.make_grid(3, n)
        bc = S.BoundarySpec.all_neumann()
        bc.set_face(2, 0, D, -1.0)
        bc.set_face(2, 1, D, 1.0)
        return g, bc, 0.0, S.Field(g), S.capacitor_sigma(g, name.split("_")[1])
    if name.startswith("trifoil_"):
        g = S.make_grid(3, n)
        return g, S.BoundarySpec.all_dirichlet(0.0), 0.0, trifoil(n)["xyz".index(name[-1])], None
    if name.startswith("deformation_"):
        g = S.make_grid(2, n)
        f, _f_raw, _ri = S.deformation_sources(circle(), g)
        if name == "deformation_circle":
            bc = S.BoundarySpec.all_neumann()
        else:
            kinds = [D, D, N, N, N, N] if name.endswith("_x") else [N, N, D, D, N, N]
            bc = S.BoundarySpec([S.FaceBc(k, 0.0) for k in kinds])
        return g, bc, 0.1, f, None
    raise KeyError(case)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("case", CASES)
def test_baseline_size_solve_matches_reference(case):
    gold = golden().get(case)
    if gold is None:
        pytest.skip(f"{case}: not in tests/golden/large.json yet (make_golden_large.py)")
    g, bc, a, f, sigma = problem(case)
    assert digest(f.numpy()) == gold["f"], "device-built source differs from the reference builder"
    if sigma is not None:
        assert digest(sigma.numpy()) == gold["sigma"]
    u = S.Field(g)
    rep = S.Solver(g, bc, a=a, sigma=sigma, config=CFG).run(f, u)
    assert [rep.converged, rep.nan_detected, rep.stagnated] == gold["flags"]
    assert [[r.cycle, r.work_units, r.residual.hex(), r.diag_min.hex()] for r in rep.rows] == gold["rows"]
    assert rep.normalization.hex() == gold["normalization"]
    assert rep.node_updates == gold["node_updates"]
    assert len(rep.trace) == gold["trace_len"]
    assert digest([t.value for t in rep.trace]) == gold["trace"]
    uh = u.numpy()
    for i, v in gold["u_samples"].items():
        assert K.bits_equal(uh[int(i)], float.fromhex(v)), i
    assert digest(uh) == gold["u"]
