"""Measure the post-solve operators (csrc/fields.cu) on one B200 against the
HBM roofline, with the reference's CPU implementation (oracle/_ref, all host
cores) timed beside them on the same inputs.

Per operator: device time of one call on resident fields (CUDA events on
the context stream, after a warm-up call, median of --reps), the algorithmic
bytes (fields read once + fields written once), achieved GB/s, fraction of
MEASURED_PEAKS.json's HBM bandwidth, and the CPU time.  Prints one JSON line
per operator.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1703_07206_b200 as S  # noqa: E402
from oracle import oracle as O  # noqa: E402  (CPU reference timing only)


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_GBps", "hbm_burst_gbs"):
            if k in d:
                return float(d[k]), "MEASURED_PEAKS.json " + k
    except (OSError, ValueError):
        pass
    return 6512.3, "bench.py measured copy bandwidth"


def timed(fn, stream, reps):
    import torch

    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    import torch

    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=9)
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--cpu-n", type=int, default=8)
    args = p.parse_args()
    peak, peak_src = hbm_peak()
    ctx = S.default_context()
    stream = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
    n = args.n
    grid = S.make_grid(3, n)
    T = grid.total
    rng = np.random.default_rng(3)
    u = S.Field.from_numpy(grid, rng.standard_normal(T))
    psi = S.VectorField.from_numpy(grid, [rng.standard_normal(T) for _ in range(3)])
    f_raw = S.Field.from_numpy(grid, np.abs(rng.standard_normal(T)) + 0.5)
    out = S.VectorField(grid)
    d = S.Field(grid)
    lib = S._capi.lib()
    from paper_1703_07206_b200.problems import _handles

    ops = {
        "curl": (lambda: lib.sgml_curl(_handles(psi.comp), _handles(out.comp)), 48),
        "gradient": (lambda: lib.sgml_gradient(u.handle, _handles(out.comp)), 32),
        "divergence": (lambda: lib.sgml_divergence(_handles(psi.comp), d.handle), 32),
        "deformation_velocity": (lambda: lib.sgml_deformation_velocity(u.handle, f_raw.handle, 1.0, 0.3,
                                                                       _handles(out.comp)), 40),
    }
    # CPU reference on a bounded sample (n = cpu_n) on all host cores
    gc = O.make_grid(3, args.cpu_n)
    cu = rng.standard_normal(gc.total)
    cpsi = rng.standard_normal((3, gc.total))
    cf = np.abs(rng.standard_normal(gc.total)) + 0.5
    cpu_ops = {
        "curl": lambda: O.curl(gc, cpsi, impl="ref"),
        "gradient": lambda: O.gradient(gc, cu, impl="ref"),
        "divergence": lambda: O.divergence(gc, cpsi, impl="ref"),
        "deformation_velocity": lambda: O.deformation_velocity(gc, cu, cf, 1.0, 0.3, impl="ref"),
    }
    have_ref = O.ref_lib() is not None
    for name, (fn, bpn) in ops.items():
        ms = timed(fn, stream, args.reps)
        gbs = bpn * T / (ms / 1e3) / 1e9
        line = {"op": name, "n": n, "N": grid.N, "ms": ms, "bytes_per_node": bpn, "achieved_gbs": gbs,
                "peak_gbs": peak, "peak_source": peak_src, "frac": gbs / peak,
                "nodes_per_s": T / (ms / 1e3)}
        if have_ref:
            t0 = time.time()
            cpu_ops[name]()
            sec = time.time() - t0
            line.update({"cpu_n": args.cpu_n, "cpu_s": sec, "cpu_nodes_per_s": gc.total / sec,
                         "cpu_threads": os.cpu_count(), "cpu_kind": "reference"})
        print(json.dumps(line), flush=True)

    # node motion (gathers) and streamlines (one thread per seed): rates only
    for steps in (10,):
        pos = S.VectorField(grid)
        fn = lambda: lib.sgml_move_nodes(u.handle, f_raw.handle, 1.0, 0.3, steps, _handles(pos.comp))  # noqa: E731
        ms = timed(fn, stream, max(2, args.reps // 2))
        line = {"op": "move_nodes", "n": n, "steps": steps, "ms": ms, "node_steps_per_s": T * steps / (ms / 1e3)}
        if have_ref:
            gm = O.make_grid(3, 6)
            t0 = time.time()
            O.move_nodes(gm, rng.standard_normal(gm.total) * 0.01, np.abs(rng.standard_normal(gm.total)) + 0.5,
                         1.0, 0.3, steps, impl="ref")
            sec = time.time() - t0
            line.update({"cpu_n": 6, "cpu_s": sec, "cpu_node_steps_per_s": gm.total * steps / sec,
                         "cpu_kind": "reference"})
        print(json.dumps(line), flush=True)
    seeds = rng.uniform(0.3, 0.7, (4096, 3))
    t0 = time.time()
    lines = S.integrate_streamlines(psi, seeds, 1e-3, 500)
    sec = time.time() - t0
    steps = sum(len(l.points) - 1 for l in lines)
    print(json.dumps({"op": "streamlines", "n": n, "seeds": len(seeds), "rk4_steps": steps, "wall_s": sec,
                      "rk4_steps_per_s": steps / sec}), flush=True)


if __name__ == "__main__":
    main()
