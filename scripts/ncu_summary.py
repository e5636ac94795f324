"""Summarise an ncu report: headline metrics + stall breakdown (debug helper)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("kernel:", d.get("Kernel Name", "")[:90])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__inst_executed.sum", "smsp__inst_executed.sum",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "launch__registers_per_thread", "sm__cycles_active.avg"]:
        if k in d:
            print("  %-70s %s %s" % (k, d[k], u[h.index(k)]))
    st = []
    for k in d:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(d[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    print("  stalls:", ", ".join("%s %.1f%%" % (k, 100 * x / tot) for x, k in sorted(st, reverse=True)[:8]))
