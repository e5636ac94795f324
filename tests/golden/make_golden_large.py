"""Reference-generated known answers at the BASELINE.json config sizes.

Run ONCE here (where /root/reference exists; hours of CPU):

    MALLOC_MMAP_THRESHOLD_=65536 OMP_NUM_THREADS=8 python tests/golden/make_golden_large.py [case ...]
    MALLOC_MMAP_THRESHOLD_=65536 OMP_NUM_THREADS=8 python tests/golden/make_golden_large.py --solves

It runs the UNMODIFIED reference solver (oracle/_ref/libsgml_ref.so, built
from /root/reference/proj/core by oracle/Makefile) on the reference's own
problem builders at the BASELINE.json configuration sizes and stores, per
case, the residual history (hex of every CycleRecord), the flags, the
normalisation, node_updates, the trace length + digest and the sha256 of
the canonical solution bits (-0.0 folded into +0.0).  Results are merged
into tests/golden/large.json after every case, so an interrupted run keeps
what it finished.  tests/test_gpu_large_parity.py solves the same problems
on the B200 (device-built inputs) and asserts all of it bit for bit.

Cases: capacitor high/low at n = 7, 8 (problems.cpp:500-521),
trifoil psi_x/psi_y/psi_z at n = 9 (problems.cpp:378-410, r = 0.14),
deformation 2049^2 (problems.cpp:302-325, CLI smoke circle) and its
mixed Dirichlet/Neumann vector-Laplace variant (two scalar solves with the
same projected source), 3D Poisson 513^3 (problems.cpp:178-193).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import cases as K  # noqa: E402
from cases import O  # noqa: E402

OUT = os.path.join(HERE, "large.json")
CFG = dict(n_r=2, tol=1e-10, max_cycles=60, safety=0.9)


def digest(a) -> str:
    return hashlib.sha256(K.canon(np.asarray(a, np.float64)).tobytes()).hexdigest()


def mixed_deformation(component: str, n: int = 11):
    """the deformation source solved as a vector Laplace
    with mixed faces -- component x: x faces Dirichlet 0, y faces Neumann;
    component y: swapped."""
    g, _b, f, s, a = O.ref_problem("deformation_circle", n)
    D, N = O.DIRICHLET, O.NEUMANN
    kinds = [D, D, N, N, N, N] if component == "x" else [N, N, D, D, N, N]
    return g, O.make_bc(kinds, [0.0] * 6), f, s, a


def problem(case: str):
    name, n = case.rsplit("@", 1)
    n = int(n)
    if name.startswith("deformation_mixed_"):
        return mixed_deformation(name[-1], n)
    if name.startswith("case:"):  # tests/cases.py solve problems
        return K.solve_problem(name[5:], n)
    if name.startswith("spec:"):  # spec:dim:n:bc:sig:a (tests/cases.py SPEC_CASES)
        _, dim, n2, bcn, sig, a = name.split(":")
        return K.spec_problem(int(dim), int(n2), bcn, sig == "1", float(a))
    return O.ref_problem(name, n)


CASES = [
    "deformation_circle@11", "deformation_mixed_x@11", "deformation_mixed_y@11",
    "capacitor_high@7", "capacitor_low@7", "capacitor_high@8", "capacitor_low@8",
    "trifoil_x@9", "trifoil_y@9", "trifoil_z@9", "poisson3d@9", "poisson3d@8",
]
# tests/golden/solves.json: the tests/cases.py solves that run the TMA
# relaxation kernels with sigma / a / Neumann / mixed faces (SOLVE_CASES_LARGE)
SOLVE_CASES = [f"case:{name}@{n}" for name, n in K.SOLVE_CASES_LARGE] + \
    [K.spec_key(*c) + f"@{c[1]}" for c in K.SPEC_CASES]


def run(case: str) -> dict:
    g, b, f, s, a = problem(case)
    # The reference's zero-weight interpolation corners on non-Dirichlet high
    # faces can read past the end of du_prev (undefined
    # behaviour).  When those bytes happen to decode as Inf/NaN the
    # reference reports nan_detected; that outcome is not the algorithm's,
    # so such a run is repeated (MALLOC_MMAP_THRESHOLD_ keeps large fields
    # in fresh, zero-tailed mappings, which makes it rare).
    for attempt in range(1, 4):
        t0 = time.time()
        res = O.solve(g, b, f, s, a, impl="ref", **CFG)
        dt = time.time() - t0
        if not res.nan_detected:
            break
    u = res.u
    mid = (g.total - 1) // 2
    return {
        "status": res.status,
        "rows": [[c, w, r.hex(), d.hex()] for c, w, r, d in res.rows],
        "trace_len": len(res.trace),
        "trace": digest([t[3] for t in res.trace]),
        "u": digest(u),
        "u_samples": {str(i): float(u[i]).hex() for i in (0, g.N + 1, mid, g.total - g.N - 2)},
        "flags": [res.converged, res.nan_detected, res.stagnated],
        "normalization": res.normalization.hex(),
        "node_updates": res.node_updates,
        "f": digest(f),
        "sigma": None if s is None else digest(s),
        "ref_seconds": round(dt, 1),
        "attempts": attempt,
        "omp_threads": int(os.environ.get("OMP_NUM_THREADS", "0") or 0),
    }


def main(argv) -> None:
    O.build(with_ref=True)
    if O.ref_lib() is None:
        raise SystemExit("reference build unavailable")
    out = OUT
    if argv[:1] == ["--solves"]:  # python make_golden_large.py --solves
        out, argv, todo = os.path.join(HERE, "solves.json"), [], SOLVE_CASES
    else:
        todo = argv or CASES
    data = json.load(open(out)) if os.path.exists(out) else {}
    for case in todo:
        if case in data and not argv:
            continue
        rec = run(case)
        data[case] = rec
        with open(out + ".tmp", "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
        os.replace(out + ".tmp", out)
        print(case, len(rec["rows"]), "cycles", rec["ref_seconds"], "s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
