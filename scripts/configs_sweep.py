"""Measure every BASELINE.json config on one B200 (plus the 1025^3 Poisson
target), with the reference CPU path sampled beside it.

For each config: the reference's own problem builder (oracle/_ref, or the
pinned C restatement for the closed-form sources), one warm-up solve, then
`--reps` timed solves (CUDA events on the engine stream, f resident in HBM);
cycles, final residual, node-updates/s (cycles * U(n, 2) * N^d / time).  The
CPU column is one reference single_cycle at the config size (or a smaller n,
stated) on all host cores.  Prints one JSON line per config.
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
from oracle import oracle as O  # noqa: E402  (builders and the CPU reference only)


def units(n):
    return O.closed_form_work_units(n, 2)


def fields(name, n):
    if name in ("sinsin2d", "poisson3d"):
        g = O.make_grid(2 if name == "sinsin2d" else 3, n)
        return g, O.all_dirichlet(0.0), O.fill(name, g), None, 0.0
    return O.ref_problem(name, n)


def gpu_run(g, b, f, s, a, reps):
    import torch

    ctx = S.Context(0)
    grid = S.make_grid(g.dim, g.n)
    bc = S.BoundarySpec([S.FaceBc(S.BcKind(b.kind[i]), b.value[i]) for i in range(6)])
    fd = S.Field.from_numpy(grid, f, ctx=ctx)
    sd = S.Field.from_numpy(grid, s, ctx=ctx) if s is not None else None
    ud = S.Field(grid, ctx=ctx)
    slv = S.Solver(grid, bc, a=a, sigma=sd, config=S.SolverConfig(n_r=2, tol=1e-10, max_cycles=60, safety=0.9),
                   ctx=ctx)
    rep = slv.run(fd, ud)  # warm-up
    stream = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.synchronize()
    e0.record(stream)
    for _ in range(reps):
        rep = slv.run(fd, ud)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    cyc = len(rep.rows)
    return {"gpu_ms": ms, "cycles": cyc, "final_residual": rep.rows[-1].residual, "converged": rep.converged,
            "node_updates_per_s": cyc * units(g.n) * g.total / (ms / 1e3),
            "footprint_gb": slv.footprint() / 1e9}


def cpu_cycle(name, n):
    g, b, f, s, a = fields(name, n)
    levels = O.sigma_levels(g, s) if s is not None else None
    t = time.time()
    O.single_cycle(g, b, f, levels, a, False, 2, 0.9, 0, 1.0, impl="ref")
    sec = time.time() - t
    return {"cpu_n": n, "cpu_cycle_s": sec, "cpu_node_updates_per_s": units(n) * g.total / sec,
            "cpu_threads": os.cpu_count()}


CONFIGS = [
    # (label, builder name, n, cpu sample n)
    ("C1 2D sin-sin 129^2", "sinsin2d", 7, 7),
    ("C1 2D poisson2d_problem(7)", "poisson2d", 7, 7),
    ("C2 3D Poisson 257^3", "poisson3d", 8, 8),
    ("C3 2D deformation 2049^2 (circle, a=0.1, all-Neumann)", "deformation_circle", 11, 11),
    ("C4 3D trifoil psi_x 513^3", "trifoil_x", 9, 8),
    ("C4 3D trifoil psi_y 513^3", "trifoil_y", 9, None),
    ("C4 3D trifoil psi_z 513^3", "trifoil_z", 9, None),
    ("3D Poisson 513^3 (bench workload)", "poisson3d", 9, None),
    ("3D Poisson 1025^3 (north-star size, 1 GPU)", "poisson3d", 10, None),
    ("C5 3D capacitor high 257^3 (sigma)", "capacitor_high", 8, None),
    ("C5 3D capacitor low 257^3 (sigma)", "capacitor_low", 8, None),
    ("C5 3D capacitor high 1025^3 (sigma)", "capacitor_high", 10, 7),
    ("C5 3D capacitor low 1025^3 (sigma)", "capacitor_low", 10, 7),
]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--only", default="")
    p.add_argument("--no-cpu", action="store_true")
    args = p.parse_args()
    for label, name, n, cpu_n in CONFIGS:
        if args.only and args.only not in label:
            continue
        t = time.time()
        g, b, f, s, a = fields(name, n)
        build_s = time.time() - t
        line = {"config": label, "builder": name, "n": n, "N": g.N, "dim": g.dim, "build_s": build_s}
        line.update(gpu_run(g, b, f, s, a, 1 if n >= 10 else args.reps))
        del f, s
        if cpu_n is not None and not args.no_cpu:
            line.update(cpu_cycle(name, cpu_n))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
