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
         e2e_single: the same through one blocking sgml_solve call per step
         (the drop-in sgml::solve path, no overlap).
  roofline  the level-0 relaxation pass (the dominant kernel), algorithmic
         bytes 24 B per relaxed node (read u_prev and g, write u; (N-2)^3
         nodes off the Dirichlet faces) / its mean launch time from CUDA
         events recorded around each launch inside the timed region;
         roofline_fp64 the same launches against the fp64 issue roof.
  cpu_baseline  the reference core itself (oracle/_ref, compiled from
         /root/reference) on the host's cores, on the SAME 513^3 problem: a
         systematic sample of the steps of its cycle (every m-th schedule
         step, m odd, ~20 s), executed through the reference's own
         restriction_into / relaxation_interpolation (oracle/ref_shim.cpp).

--impl reference: the reference's CPU solve of the same 513^3 problem on all
host cores, one full cycle (its schedule steps plus the residual recurrence,
exactly as solve() runs cycle 0) split into K consecutive timed chunks, one
chunk per step; value = the cycle's node updates / the K chunks' time.  The
reference's cost per cycle does not depend on the cycle index, so this is
its solve rate; the full 8-cycle 513^3 solve takes ~8x the cycle.
Multi-GPU (--gpus N > 1): without torchrun the script re-launches itself
under torch.distributed.run with N ranks (exit 2 if fewer GPUs are
visible); the N ranks solve the same 513^3 problem with the z-slab
decomposition (one NCCL clique, halo planes between
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
    # (--grid-n: the spelling that survives torch.distributed.run's option
    # matching, which reads a bare --n as an abbreviation of its own options)
    p.add_argument("--n", "--grid-n", dest="n", type=int, default=9, help="grid exponent, N = 2^n + 1 (default 513^3)")
    p.add_argument("--engine", choices=["compact", "literal"], default="compact")
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

def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def ref_session(n: int):
    """The reference's solve of the bench problem, steppable (oracle/ref_shim.cpp)."""
    from oracle import oracle as O  # checker / baseline only
    g = O.make_grid(3, n)
    sess = O.RefSession(g, O.all_dirichlet(0.0), poisson3d_source(n), None, 0.0, 2, 0.9)
    return O, g, sess


def chunk_plan(schedule, k: int):
    """Split one cycle's schedule steps into min(k, steps) consecutive chunks
    of about equal work units."""
    from oracle import oracle as O
    w = [O.RefSession.units(st) for st in schedule]
    U = sum(w)
    k = max(1, min(k, len(schedule)))
    chunks, cur, acc = [], [], 0
    for i, wi in enumerate(w):
        cur.append(i)
        acc += wi
        left_steps = len(w) - i - 1
        left_chunks = k - len(chunks) - 1
        if left_chunks > 0 and (acc >= U * (len(chunks) + 1) / k or left_steps == left_chunks):
            chunks.append(cur)
            cur = []
    chunks.append(cur)
    return chunks, w, U


def ref_threads() -> int:
    """OpenMP threads for the reference's loops: every host core.  Under
    torch.distributed.run, which sets OMP_NUM_THREADS=1 for each process, the
    reference runs on rank 0 alone and takes all cores back (must run before
    the reference build is loaded)."""
    omp = os.environ.get("OMP_NUM_THREADS", "")
    if not omp or (int(os.environ.get("WORLD_SIZE", "1")) > 1 and omp == "1"):
        os.environ["OMP_NUM_THREADS"] = str(host_cores())
    return int(os.environ["OMP_NUM_THREADS"])


def cpu_sample(n: int, budget_s: float = 20.0):
    """cpu_baseline: the reference core (oracle/_ref) on the same problem, a
    systematic sample of its cycle's schedule steps (every m-th step, m odd so
    both step kinds are sampled) sized for ~budget_s; the C port's single
    cycles at 129^3 if the reference build is absent."""
    cores = ref_threads()  # the threads the reference's OpenMP loops use
    from oracle import oracle as O  # checker / baseline only
    if O.ref_lib() is None:
        g = O.make_grid(3, 7)
        f = O.fill("poisson3d", g)
        t0 = time.perf_counter()
        st, _, _, w = O.single_cycle(g, O.all_dirichlet(0.0), f, None, 0.0, False, 2, 0.9, 0, 1.0, impl="c")
        dt = time.perf_counter() - t0
        return (units(7) * g.total / dt, "port", 1,
                f"1 x single_cycle of poisson3d_problem(7) (129^3) by the C restatement, 1 thread, {dt:.1f} s")
    _, g, sess = ref_session(n)
    sched = sess.schedule
    U = units(n)
    est_s = U * g.total / 3e8  # rough reference rate on ~16 cores
    m = max(1, int(round(est_s / budget_s)))
    if m % 2 == 0:
        m += 1
    picks = list(range(0, len(sched), m))
    sess.begin_cycle(False)
    t_total, done = 0.0, 0
    for i in picks:
        t0 = time.perf_counter()
        assert sess.step(i) == 0
        t_total += time.perf_counter() - t0
        done += O.RefSession.units(sched[i])
    sess.close()
    rate = done * g.total / t_total
    sample = (f"reference solve of poisson3d_problem({n}) ({g.N}^3): every {m}-th of the {len(sched)} "
              f"schedule steps of its cycle ({len(picks)} steps, {done} of {U} work units) on {cores} "
              f"OpenMP threads, {t_total:.1f} s")
    return rate, "reference", cores, sample, t_total


def run_reference(args, dist):
    """--impl reference: the reference's CPU solve of the same problem on this
    box's host cores, one full cycle in K consecutive chunks (one per step)."""
    if dist.rank != 0:
        return None
    cores = ref_threads()
    O, g, sess = ref_session(args.n)
    chunks, w, U = chunk_plan(sess.schedule, args.steps)
    T = g.total

    def run_chunk(c: int) -> float:
        t0 = time.perf_counter()
        if c == 0:
            sess.begin_cycle(False)
        for i in chunks[c]:
            if sess.step(i) != 0:
                raise RuntimeError("reference pass failed")
        if c == len(chunks) - 1:
            sess.recurrence()
        return time.perf_counter() - t0

    for i in range(args.warmup):
        run_chunk(i % len(chunks))
    secs, work = [], 0
    for i in range(args.steps):
        c = i % len(chunks)
        secs.append(run_chunk(c))
        work += sum(w[j] for j in chunks[c])
    sess.close()
    total_s = sum(secs)
    value = work * T / total_s
    cycle_s = total_s * U / work
    sample = (f"cycle 0 of the reference solve of poisson3d_problem({args.n}) ({g.N}^3, U={U} work units, "
              f"{len(sess.schedule)} schedule steps + the residual recurrence) split into {len(chunks)} "
              f"consecutive chunks, one per step; {cores} OpenMP threads")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"3D Poisson {g.N}^3 fp64, Dirichlet 0, manufactured "
                               f"sin(pi x)sin(pi y)sin(pi z) (poisson3d_problem({args.n})), "
                               "solve to 1e-10 normalised residual",
                   "n": args.n, "N": g.N, "n_r": 2, "tol": 1e-10, "safety": 0.9,
                   "sample": "one full cycle of the solve (every cycle costs the same)"},
        "cycle_s": cycle_s,
        "time_to_tol_s_est": 8 * cycle_s,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
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
        # the single-call drop-in path: sgml::solve(ProblemSpec) -> one blocking
        # sgml_solve per step on pageable host memory (std::vector-like numpy
        # arrays), no overlap between steps
        fpg = np.ascontiguousarray(f_host)
        upg = np.empty(T, np.float64)

        def call_pageable():
            rbuf.c.n_rows = rbuf.c.n_trace = 0
            _capi.check(lib.sgml_solve(ctx.handle, 3, n, C.byref(cbc), fpg.ctypes.data_as(_capi._D), None, 0.0,
                                       C.byref(ccfg), C.byref(copts), upg.ctypes.data_as(_capi._D),
                                       C.byref(rbuf.c)))
            return rbuf.c.n_rows

        call_pageable()
        k1 = min(args.steps, 5)
        dist.barrier()
        t_0 = time.perf_counter()
        cyc1 = sum(call_pageable() for _ in range(k1))
        dt1 = dist.reduce(time.perf_counter() - t_0, "max")
        e2e["single_call"] = {"value": cyc1 * units(n) * T / dt1, "unit": UNIT, "steps": k1,
                              "ms_per_step": 1e3 * dt1 / k1, "h2d_bytes_per_step": nbytes,
                              "d2h_bytes_per_step": nbytes,
                              "api": "sgml_solve per step (the sgml::solve drop-in path), pageable host f/u, "
                                     "host wall clock around the blocking call"}

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
            rate, kind, cores, sample, _ = cpu_sample(args.n)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                                    "sample": sample}
        except Exception as exc:  # the baseline must not sink the measurement
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": None,
                                    "sample": f"unavailable: {exc}"}
    return line if dist.rank == 0 else None


def visible_gpus() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launcher_cmd(gpus: int, argv) -> list:
    """The torch.distributed.run command that runs this script on `gpus` ranks
    of this node (one process per GPU)."""
    # (a bare --n would be read by torch.distributed.run as one of its own
    # options: pass it on as --grid-n)
    argv = ["--grid-n" if a == "--n" else ("--grid-n=" + a[4:] if a.startswith("--n=") else a) for a in argv]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]


def main():
    args = parse()
    world, rank, local = dist_env()
    if world == 1 and args.gpus > 1 and args.impl == "ours":
        # --gpus N without torchrun: one process per GPU, or fail loudly (a
        # single process must never report an N-GPU number)
        have = visible_gpus()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
                  file=sys.stderr, flush=True)
            sys.exit(2)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout one JSON line
        cmd = launcher_cmd(args.gpus, sys.argv[1:])
        os.execv(cmd[0], cmd)
    if world > 1:
        args.gpus = world
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if args.impl == "ours" and visible_gpus() < world:
            print(f"bench.py: {world} ranks need {world} visible GPUs, found {visible_gpus()}",
                  file=sys.stderr, flush=True)
            sys.exit(2)
    # (the reference arm runs on rank 0's host cores alone and needs neither a
    # GPU per rank nor a process group: the other ranks exit at once)
    dist = Dist(world if args.impl == "ours" else 1, rank, local)
    try:
        line = run_reference(args, dist) if args.impl == "reference" else run_ours(args, dist)
        if line is not None:
            print(json.dumps(line), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
