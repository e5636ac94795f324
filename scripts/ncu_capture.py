"""ncu evidence for the 513^3 solve, selected by kernel NAME and GRID (not by a
launch-skip count that drifts when the schedule changes).  Run on the GPU box:

    python scripts/ncu_capture.py --n 9 --out gpurun_out/r02

1. Launch list of one solve (scripts/prof_solve.py n 1) with
   gpu__time_duration.sum / launch__grid_size / registers  ->  <out>_launches.csv
2. Targets picked from that list by full template name + grid size:
   relax0 (level-0 pass), relax1 (level-1 pass with du), residual, sigma relax0
   (capacitor problem), materialise at level 0 with chains of 8 / 4 / 1
   entries, pyramid 0 -> 1, the one-CTA small-level kernel.
3. One `ncu --set full --import-source on` capture per target (-k <base name>
   --launch-skip <ordinal among that base name's launches> -c 1), summarised
   into <out>_ncu_<label>.txt; the summary asserts the captured kernel's
   template name and grid equal the target's.
"""
from __future__ import annotations

import argparse
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "scripts", "prof_solve.py")

SUMMARY_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__cycles_active.avg",
]


def run(cmd, **kw):
    print("+", " ".join(cmd), flush=True)
    return subprocess.run(cmd, check=True, **kw)


def read_ncu_csv(path):
    """Rows of an ncu --csv log (skipping ==PROF== lines) as dicts, one per
    (kernel ID, metric)."""
    text = open(path).read()
    start = text.find('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def launch_list(n, out, problem, count=None):
    path = out + f"_launches_{problem}.csv"
    lim = ["--launch-count", str(count)] if count else []
    run(["ncu", "--metrics", "gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread",
         "--clock-control", "none", *lim, "--csv", "--log-file", path, sys.executable, PROF, str(n), "1", "compact",
         problem])
    launches = {}
    for r in read_ncu_csv(path):
        k = int(r["ID"])
        d = launches.setdefault(k, {"id": k, "name": r["Kernel Name"]})
        d[r["Metric Name"]] = r["Metric Value"].replace(",", "")
    return [launches[k] for k in sorted(launches)], path


def base(name):
    """k_relax_tma from 'void unnamed>::k_relax_tma<3, 0, ...>(...)'."""
    return name.split("<")[0].split("(")[0].strip().split(" ")[-1].split("::")[-1]


def pick(launches, name_part, nth=0, largest=True):
    """The nth launch (in order) whose full name contains name_part, among those
    with the largest grid if `largest`; returns (launch, ordinal among its base
    name's launches)."""
    cand = [L for L in launches if name_part in L["name"]]
    if not cand:
        return None, None
    if largest:
        g = max(int(L["launch__grid_size"]) for L in cand)
        cand = [L for L in cand if int(L["launch__grid_size"]) == g]
    if nth >= len(cand):
        return None, None
    L = cand[nth]
    b = base(L["name"])
    ordinal = [M["id"] for M in launches if base(M["name"]) == b].index(L["id"])
    return L, ordinal


def summarize(rep, target, label, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    if len(r) < 3:
        raise SystemExit(f"{label}: no kernel captured in {rep}")
    h, u, v = r[0], r[1], r[2]
    name = v[h.index("Kernel Name")]
    grid = v[h.index("launch__grid_size")].replace(",", "") if "launch__grid_size" in h else "?"
    ok = name == target["name"] and grid == target["launch__grid_size"]
    lines = [f"label: {label}", f"kernel: {name}", f"grid: {grid}",
             f"selection check (name and grid equal the launch-list target): {'OK' if ok else 'MISMATCH'}"]
    for m in SUMMARY_METRICS:
        if m in h:
            i = h.index(m)
            lines.append(f"  {m:70s} {v[i]:>18s} {u[i]}")
    st = []
    for i, m in enumerate(h):
        if m.startswith("smsp__average_warps_issue_stalled") and m.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), m.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    tot = sum(a for a, _ in st) or 1.0
    lines.append("  stalls: " + ", ".join(f"{b} {100 * a / tot:.1f}%" for a, b in sorted(st, reverse=True)[:8]))
    txt = "\n".join(lines) + "\n"
    with open(f"{out}_ncu_{label}.txt", "w") as fh:
        fh.write(txt)
    print(txt, flush=True)
    if not ok:
        raise SystemExit(f"{label}: captured kernel differs from the target")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=9)
    ap.add_argument("--out", default="gpurun_out/r02")
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", default="/tmp/ncu_reps", help="where the .ncu-rep files go (large)")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    os.makedirs(args.reps, exist_ok=True)
    launches, _ = launch_list(args.n, args.out, "poisson")
    sig_launches = []
    if not args.only or "sigma" in args.only:
        sig_launches, _ = launch_list(args.n, args.out, "capacitor", count=1500)  # (cycle 0 is enough)
    T = [  # label, name part, nth, largest, launch list
        ("relax0", "k_relax_tma<3, 0, 0, 0, 0, 0>", 0, True, launches, "poisson"),
        ("relax1", "k_relax_tma<3, 0, 0, 0, 1, 0>", 0, True, launches, "poisson"),
        ("residual", "k_relax_tma<3, 0, 0, 1, 1, 0>", 0, True, launches, "poisson"),
        ("mat0_c8", "k_materialize4<3, 2, 0>", 0, True, launches, "poisson"),
        ("mat0_c4", "k_materialize4<3, 2, 0>", 4, True, launches, "poisson"),
        ("mat0_c1", "k_materialize4<3, 2, 0>", 7, True, launches, "poisson"),
        ("matl0_c8", "k_materialize_l0<3>", 0, True, launches, "poisson"),
        ("matl0_c4", "k_materialize_l0<3>", 4, True, launches, "poisson"),
        ("matl0_c1", "k_materialize_l0<3>", 7, True, launches, "poisson"),
        ("pyramid01", "k_pyramid_ext<3>", 0, True, launches, "poisson"),
        ("small", "k_relax_small<3, 0, 0>", 0, True, launches, "poisson"),
        ("sigma_relax0", "k_relax_tma<3, 1, 0, 0, 0, 0>", 0, True, sig_launches, "capacitor"),
    ]
    for label, part, nth, largest, L, problem in T:
        if args.only and label not in args.only.split(","):
            continue
        target, ordinal = pick(L, part, nth, largest)
        if target is None:
            print(f"{label}: no launch matches {part!r}", flush=True)
            continue
        rep = os.path.join(args.reps, f"{os.path.basename(args.out)}_{label}")
        run(["ncu", "--set", "full", "--import-source", "on", "--clock-control", "none", "-k", "regex:" + base(target["name"]),
             "--launch-skip", str(ordinal), "--launch-count", "1", "-f", "-o", rep,
             sys.executable, PROF, str(args.n), "1", "compact", problem], stdout=subprocess.DEVNULL)
        summarize(rep + ".ncu-rep", target, label, args.out)


if __name__ == "__main__":
    main()
