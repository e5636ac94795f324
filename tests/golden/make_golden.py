"""Generate the golden vectors from the UNMODIFIED reference core.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/libsgml_ref.so from the reference sources in place
(oracle/Makefile), runs the reference on the deterministic inputs of
tests/cases.py and writes:

  tests/golden/golden.json   per-case sha256 of the canonical result bits
                             (-0.0 folded to +0.0) plus scalars (diag, rows)
  tests/golden/arrays.npz    full result arrays for a few small 2D cases

tests/test_oracle_pinning.py checks the C restatement (oracle/) against
these files on any host, and tests/test_gpu_parity.py checks the B200
kernels against the restatement.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import cases as K  # noqa: E402
from cases import O  # noqa: E402


def digest(a) -> str:
    return hashlib.sha256(K.canon(np.asarray(a, np.float64)).tobytes()).hexdigest()


def key(*parts) -> str:
    return "/".join(str(p) for p in parts)


def main() -> None:
    O.build(with_ref=True)
    if O.ref_lib() is None:
        raise SystemExit("reference build unavailable")
    out = {"relax": {}, "restriction": {}, "residual": {}, "solve": {}, "schedule": {}, "fields": {}}
    arrays = {}

    for case in K.relax_cases(full=False):
        dim, n, level, bcn, sig, a, hom = case
        g, b, up, dup, gs, s = K.relax_inputs(*case)
        st, u, du, diag = O.relax(g, b, up, dup, level, gs, s, a, 0.9, hom, impl="ref")
        k = key(dim, n, level, bcn, int(sig), a, int(hom))
        out["relax"][k] = {"status": st, "diag": diag.hex(), "u": digest(u), "du": digest(du)}
        if dim == 2 and not sig and a == 0.0:
            arrays["relax_u/" + k] = u
            arrays["relax_du/" + k] = du

    for dim, n in ((2, 4), (3, 3)):
        g = O.make_grid(dim, n)
        f = O.lcg(g, 11 + dim)
        for bcn in ("dir0", "neumann", "dir_distinct", "low_dir_high_neu"):
            for v in range(0, n + 1):
                r, w = O.restriction(g, K.bc(bcn), f, v, impl="ref")
                k = key(dim, n, bcn, v)
                out["restriction"][k] = {"work": w, "out": digest(r)}
                if dim == 2:
                    arrays["restriction/" + k] = r

    for dim, n in ((2, 4), (3, 3)):
        g = O.make_grid(dim, n)
        e = O.lcg(g, 23)
        f = O.lcg(g, 29)
        for bcn in ("dir0", "neumann", "dir_distinct", "low_dir_high_neu"):
            for sig in (False, True):
                for a in (0.0, 0.3):
                    s = K.sigma_field(g, 31) if sig else None
                    r = O.residual_update(g, K.bc(bcn), f, e, s, a, impl="ref")
                    out["residual"][key(dim, n, bcn, int(sig), a)] = {"r": digest(r)}

    for name, n in K.SOLVE_CASES:
        g, b, f, s, a = K.solve_problem(name, n)
        res = O.solve(g, b, f, s, a, n_r=2, tol=1e-10, max_cycles=40, impl="ref")
        out["solve"][key(name, n)] = {
            "status": res.status,
            "rows": [[c, w, r.hex(), d.hex()] for c, w, r, d in res.rows],
            "trace": digest([t[3] for t in res.trace]),
            "trace_len": len(res.trace),
            "u": digest(res.u),
            "flags": [res.converged, res.nan_detected, res.stagnated],
            "normalization": res.normalization.hex(),
            "node_updates": res.node_updates,
        }

    for n in range(1, 11):
        for n_r in (1, 2, 3, 8):
            out["schedule"][key(n, n_r)] = int(O.ref_lib().ref_closed_form_work_units(n, n_r))

    for dim, n in K.FIELD_GRIDS:
        d = K.field_inputs(dim, n)
        g = d["g"]
        rec = {"gradient": digest(O.gradient(g, d["u"], impl="ref")),
               "divergence": digest(O.divergence(g, d["v"], impl="ref"))}
        if dim == 3:
            rec["curl"] = digest(O.curl(g, d["psi"], impl="ref"))
        st, vel = O.deformation_velocity(g, d["u"], d["f_raw"], d["raw_integral"], d["t"], impl="ref")
        rec["deformation_velocity"] = [st, digest(vel)]
        st, pos = O.move_nodes(g, 0.01 * d["u"], d["f_raw"], d["raw_integral"], d["t"], d["steps"], impl="ref")
        rec["move_nodes"] = [st, digest(pos)]
        lines = []
        for field in ("swirl", "v"):
            for seed in d["seeds"]:
                pts, stop = O.integrate_streamline(g, d[field], seed, d["step"], d["max_steps"], impl="ref")
                lines.append([field, len(pts), stop, digest(pts)])
        rec["streamlines"] = lines
        rec["sample"] = [digest(O.sample_vector(g, d["v"], p, impl="ref")) for p in d["seeds"]]
        out["fields"][key(dim, n)] = rec

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "arrays.npz"), **arrays)
    print("relax", len(out["relax"]), "restriction", len(out["restriction"]), "residual",
          len(out["residual"]), "solve", len(out["solve"]), "fields", len(out["fields"]), "arrays", len(arrays))


if __name__ == "__main__":
    main()
