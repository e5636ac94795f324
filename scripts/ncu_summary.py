"""One-screen summary of an ncu --set full report (raw page): duration, DRAM
bytes, fp64 pipe, issue, occupancy, registers and the top stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
print("kernel:", v[h.index("Kernel Name")][:120])
for m in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
          "sm__cycles_active.avg"]:
    if m in h:
        i = h.index(m)
        print(f"  {m:70s} {v[i]:>16s} {u[i]}")
st = []
for i, m in enumerate(h):
    if m.startswith("smsp__average_warps_issue_stalled") and m.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v[i]), m.split("stalled_")[1].split("_per")[0]))
        except ValueError:
            pass
tot = sum(a for a, _ in st)
print("  stalls: " + ", ".join(f"{b} {100 * a / tot:.1f}%" for a, b in sorted(st, reverse=True)[:8]))
