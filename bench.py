#!/usr/bin/env python
"""bench.py — BASELINE.json metric: fp64 node-updates/s & time-to-1e-10 residual.

Workload (N = 1): the reference's 3D Poisson problem at 513^3
(poisson3d_problem(9): f = -3 pi^2 sin(pi x) sin(pi y) sin(pi z), Dirichlet 0),
solved to a 1e-10 normalised residual with SolverConfig{n_r=2, safety=0.9}.
One step = one complete solve (every cycle, the residual recurrence and the
convergence test).  node-updates/s uses the reference's own accounting,
cycles * U(n, n_r) * N^3 / time (cycle.cpp:191-192, sgml_main.cpp:218-219).

  value  device time of K solves with f already resident in HBM (CUDA events
         on the engine's stream); every field is 1.08 GB, far above the 126 MB L2.
  e2e    the C-ABI with pinned host buffers: every step copies its f in
         (H2D), solves, and copies its u out (D2H) inside the timed region
         (sgml_solve_many: step k+1's H2D and step k-1's D2H overlap step k).
  roofline  the level-0 relaxation pass (the dominant kernel), algorithmic
         bytes 24 B per relaxed node (read u_prev and g, write u; (N-2)^3
         nodes off the Dirichlet faces) / its mean launch time from CUDA
         events recorded around each launch inside the timed region;
         roofline_fp64 the same launches against the fp64 issue roof.
  cpu_baseline  the reference core itself (oracle/_ref, compiled from
         /root/reference) on the host's cores, one single_cycle of
         poisson3d_problem(7) (129^3) per sample.

--impl reference runs only that CPU reference (rank 0) on the same metric.
Multi-GPU (torchrun, N > 1): the N ranks solve the same 513^3 problem with
the z-slab decomposition (one NCCL clique, halo planes between
neighbours, max reductions; strong scaling, value = the problem's updates /
the max-over-ranks device time).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")
METRIC = "fp64 node-updates/s (3D Poisson solve to 1e-10)"
UNIT = "node-updates/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=9, help="grid exponent, N = 2^n + 1 (default 513^3)")
    p.add_argument("--engine", choices=["compact", "literal"], default="compact")
    p.add_argument("--cpu-n", type=int, default=7, help="grid exponent of the CPU sample")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


# ------------------------------------------------------------------ env ----

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Dist:
    """torch.distributed plumbing (barrier, max/sum over ranks); no-op at N = 1."""

    def __init__(self, world: int, rank: int, local: int):
        self.world, self.rank, self.local = world, rank, local
        self.pg = None
        if world > 1:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(local)
            dist.init_process_group(backend=backend)
            self.dist, self.torch, self.backend = dist, torch, backend

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def reduce(self, x: float, op: str) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device=f"cuda:{self.local}" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


class Clocks:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------- workload ----

def poisson3d_source(n: int) -> np.ndarray:
    """poisson3d_problem(n) source (problems.cpp:178-193), x-fastest order."""
    N = (1 << n) + 1
    h = 1.0 / (N - 1)
    s = np.sin(np.pi * (np.arange(N) * h))
    c = -3.0 * np.pi * np.pi
    f = np.empty((N, N, N), np.float64)
    for k in range(N):
        f[k] = c * (np.outer(s, s) * s[k])   # ((sx*sy)*sz), then * (-3 pi) * pi
    return f.reshape(-1)


def units(n: int, n_r: int = 2) -> int:
    tot = 0
    for v1 in range(n):
        tot += v1 * (v1 + 1) // 2 + (v1 + 1) * min(n_r, 2 ** (n - v1))
    return tot + min(n_r, 2 ** n)


# ------------------------------------------------------------ cpu side ----

def cpu_sample(n: int, budget_s: float = 12.0):
    """The reference core (oracle/_ref) or, if absent, the C port: single cycles
    of poisson3d at 2^n+1 until ~budget_s; returns (rate, kind, cores, sample)."""
    from oracle import oracle as O  # checker / baseline only
    impl = "ref" if O.ref_lib() is not None else "c"
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    g = O.make_grid(3, n)
    f = O.fill("poisson3d", g)
    bc = O.all_dirichlet(0.0)
    t_total, cycles = 0.0, 0
    while cycles < 1 or (t_total < budget_s and cycles < 30):
        t0 = time.perf_counter()
        st, _, _, w = O.single_cycle(g, bc, f, None, 0.0, False, 2, 0.9, 0, 1.0, impl=impl)
        t_total += time.perf_counter() - t0
        cycles += 1
        assert st == 0 and w == units(n)
    rate = cycles * units(n) * g.total / t_total
    kind = "reference" if impl == "ref" else "port"
    sample = (f"{cycles} x single_cycle of poisson3d_problem({n}) ({g.N}^3, U={units(n)} passes) "
              f"on {cores} OpenMP threads, {t_total:.1f} s")
    return rate, kind, cores, sample, t_total / cycles


def run_reference(args, dist):
    """--impl reference: the reference's CPU path on this box's host cores."""
    if dist.rank != 0:
        return None
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    rates, secs = [], []
    for i in range(args.warmup + args.steps):
        rate, kind, cores, sample, sec = cpu_sample(args.cpu_n, budget_s=0.0)
        if i >= args.warmup:
            rates.append(rate)
            secs.append(sec)
    value = statistics.median(rates)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"3D Poisson {(1 << args.n) + 1}^3 fp64 solve to 1e-10 "
                               f"(sampled: one reference cycle per step at {(1 << args.cpu_n) + 1}^3)",
                   "n": args.n, "sample_n": args.cpu_n, "n_r": 2, "tol": 1e-10, "safety": 0.9},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------- gpu side ----

def run_ours(args, dist):
    import torch

    import paper_1703_07206_b200 as S
    from paper_1703_07206_b200 import _capi

    dev = dist.local
    ctx = S.Context(dev)
    from paper_1703_07206_b200.dist import join_torch_clique
    join_torch_clique(ctx)  # N > 1: z-slab clique over NCCL
    n = args.n
    grid = S.make_grid(3, n)
    T = grid.total
    f_host = poisson3d_source(n)
    bc = S.BoundarySpec.all_dirichlet(0.0)
    cfg = S.SolverConfig(n_r=2, tol=1e-10, max_cycles=60, safety=0.9)
    # the timed region instruments only the level-0 relaxation launches (the
    # roofline kernel); the full per-class breakdown comes from one extra,
    # separately instrumented solve after it
    opts = S.SolverOptions(engine=args.engine, timing=True, timing_classes=1 << 0)
    f_dev = S.Field.from_numpy(grid, f_host, ctx=ctx)
    u_dev = S.Field(grid, ctx=ctx)
    solver = S.Solver(grid, bc, config=cfg, options=opts, ctx=ctx)

    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{dev}")
    for _ in range(args.warmup):
        rep = solver.run(f_dev, u_dev)
    cycles = len(rep.rows)

    # ---- timed region: K solves, inputs resident in HBM ----------------
    reps = []
    dist.barrier()
    torch.cuda.synchronize(dev)
    ctx.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            rb = solver.run(f_dev, u_dev)
            reps.append(rb)
        e1.record(stream)
        e1.synchronize()
    ctx.synchronize()
    torch.cuda.synchronize(dev)
    dist.barrier()
    ms_local = e0.elapsed_time(e1)
    ms = dist.reduce(ms_local, "max")
    cyc_total = sum(len(r.rows) for r in reps)
    updates_local = cyc_total * units(n) * T
    updates = float(updates_local)  # one problem, solved jointly by the N ranks
    value = updates / (ms / 1e3)
    launches = sum(r.kernel_launches for r in reps)

    # relax0 launch time from the engine's own events inside the timed region
    # (same stream; the last solve's report)
    lib = _capi.lib()
    rb = solver._rb.c
    relax0_ms = rb.class_ms[0] / max(1, rb.class_launches[0])
    # per-class breakdown: one extra solve with every class instrumented
    full = S.Solver(grid, bc, config=cfg, options=S.SolverOptions(engine=args.engine, timing=True), ctx=ctx)
    full.run(f_dev, u_dev)
    rf = full._rb.c
    cls = {name: {"ms_per_solve": rf.class_ms[k], "launches_per_solve": int(rf.class_launches[k])}
           for k, name in enumerate(_capi.CLASS_NAMES[:7])}
    cls["note"] = "one separately instrumented solve (events around every launch)"
    del full
    # the pass covers the nodes off the Dirichlet faces ((N-2)^3 here); the
    # face nodes keep their value and are not touched
    relaxed = float((grid.N - 2) ** 3)
    bytes_per_launch = 24.0 * relaxed
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = bytes_per_launch / (relax0_ms / 1e3) / 1e9
    # the same launches against the fp64 issue roof: 76 fp64 operations per
    # relaxed node (26 differences, 20 weight products, 25 chain adds,
    # op / Euler step 5); 62 DADD/clk/SM measured x 148 SMs x 1.965 GHz
    fp64_ops = 76.0 * relaxed
    fp64_peak = 62.0 * 148 * 1.965e9
    traffic = None
    if os.path.exists(TRAFFIC_PATH):
        traffic = json.load(open(TRAFFIC_PATH)).get("relax0_bytes_per_launch", {}).get(str(n))

    # ---- e2e: drop-in sgml_solve with pinned host buffers --------------
    e2e = None
    if not args.no_e2e:
        nbytes = T * 8
        fp, up = C.c_void_p(), C.c_void_p()
        _capi.check(lib.sgml_host_alloc(nbytes, C.byref(fp)))
        _capi.check(lib.sgml_host_alloc(nbytes, C.byref(up)))
        fh = np.frombuffer((C.c_double * T).from_address(fp.value), np.float64)
        fh[:] = f_host
        rbuf = S.api._ReportBuffers()
        copts = S.SolverOptions(engine=args.engine).to_c()
        ccfg = cfg.to_c()
        cbc = bc.to_c()

        def call():
            rbuf.c.n_rows = rbuf.c.n_trace = 0
            _capi.check(lib.sgml_solve(ctx.handle, 3, n, C.byref(cbc), C.cast(fp, _capi._D), None, 0.0,
                                       C.byref(ccfg), C.byref(copts), C.cast(up, _capi._D),
                                       C.byref(rbuf.c)))
            return rbuf.c.n_rows

        call()  # builds the cached engine
        # the timed steps go through sgml_solve_many: every step still copies
        # its f in and its u out (pinned host buffers), but step k+1's H2D and
        # step k-1's D2H overlap step k's solve on a copy stream
        e2e_reps = (_capi.Report * args.steps)()
        rbufs = [S.api._ReportBuffers() for _ in range(args.steps)]
        for i, rb in enumerate(rbufs):
            e2e_reps[i] = rb.c
        fptrs = (_capi._D * args.steps)(*[C.cast(fp, _capi._D)] * args.steps)
        uptrs = (_capi._D * args.steps)(*[C.cast(up, _capi._D)] * args.steps)
        # one untimed pipelined call allocates the second staging buffers
        _capi.check(lib.sgml_solve_many(ctx.handle, 3, n, C.byref(cbc), 1, fptrs, None, 0.0,
                                        C.byref(ccfg), C.byref(copts), uptrs, e2e_reps))
        for i, rb in enumerate(rbufs):
            e2e_reps[i] = rb.c
        dist.barrier()
        ctx.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        _capi.check(lib.sgml_solve_many(ctx.handle, 3, n, C.byref(cbc), args.steps, fptrs, None, 0.0,
                                        C.byref(ccfg), C.byref(copts), uptrs, e2e_reps))
        t1.record(stream)
        t1.synchronize()
        e2e_cycles = sum(int(r.n_rows) for r in e2e_reps)
        e2e_last = e2e_reps[args.steps - 1]
        e2e_final = float(e2e_last.rows[e2e_last.n_rows - 1].residual) if e2e_last.n_rows else None
        e2e_ms = dist.reduce(t0.elapsed_time(t1), "max")
        e2e_updates = float(e2e_cycles * units(n) * T)
        uh = np.frombuffer((C.c_double * T).from_address(up.value), np.float64)
        e2e_ok = bool(np.isfinite(uh).all())
        e2e = {"value": e2e_updates / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": e2e_ms / args.steps,
               "api": "sgml_solve_many (C-ABI, pinned host f/u; transfers of neighbouring steps overlap)",
               "finite": e2e_ok, "final_residual": e2e_final}
        lib.sgml_host_free(fp)
        lib.sgml_host_free(up)

    last = reps[-1]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3D Poisson {grid.N}^3 fp64, Dirichlet 0, manufactured "
                               f"sin(pi x)sin(pi y)sin(pi z) (poisson3d_problem({n})), "
                               "solve to 1e-10 normalised residual",
                   "n": n, "N": grid.N, "n_r": 2, "tol": 1e-10, "safety": 0.9,
                   "engine": args.engine,
                   "parallelism": "single" if args.gpus == 1 else f"zslab{args.gpus}",
                   "l2": "inputs larger than L2 (1.08 GB per field vs 126 MB)"},
        "time_to_tol_s": ms / args.steps / 1e3,
        "cycles": cycles,
        "final_residual": last.rows[-1].residual if last.rows else None,
        "converged": last.converged,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "relax0 (k_relax_tma<3,0,0,0,0>, level-0 relaxation pass)",
                     "bytes_per_launch": bytes_per_launch, "mean_launch_ms": relax0_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
        "roofline_fp64": {"achieved": fp64_ops / (relax0_ms / 1e3), "peak": fp64_peak,
                          "unit": "fp64 ops/s", "frac": fp64_ops / (relax0_ms / 1e3) / fp64_peak,
                          "ops_per_node": 76,
                          "peak_source": "scripts/micro/dp_latency.cu: 62 DADD/clk/SM at 1965 MHz"},
        "kernels": cls,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if not args.no_cpu and dist.rank == 0 and args.gpus == 1:
        try:
            rate, kind, cores, sample, _ = cpu_sample(args.cpu_n)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                                    "sample": sample}
        except Exception as exc:  # the baseline must not sink the measurement
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": None,
                                    "sample": f"unavailable: {exc}"}
    return line if dist.rank == 0 else None


def main():
    args = parse()
    world, rank, local = dist_env()
    if world > 1:
        args.gpus = world
    dist = Dist(world, rank, local)
    try:
        line = run_reference(args, dist) if args.impl == "reference" else run_ours(args, dist)
        if line is not None:
            print(json.dumps(line), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
