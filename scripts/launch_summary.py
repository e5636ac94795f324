"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum[,...] --csv`,
one row per (launch, metric)) by kernel and grid shape: for the level kernels
the grid identifies the level.  usage: launch_summary.py <launches.csv>"""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read()
text = text[text.find('"ID"'):]
launches = {}
for r in csv.DictReader(io.StringIO(text)):
    d = launches.setdefault(int(r["ID"]), {"name": r["Kernel Name"], "grid": r["Grid Size"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for d in launches.values():
    name = d["name"].split("(")[0].replace("unnamed>::", "").replace("void ", "")
    key = f"{name} grid{d['grid']}" if ("k_relax_tma" in name or "k_materialize" in name) else name
    tot[key] += d["gpu__time_duration.sum"] * 1e-6
    cnt[key] += 1
all_ms = sum(tot.values())
print(f"{len(launches)} launches, {all_ms:.1f} ms total (serialised, cold-cache ncu timings)")
print(f"{'kernel':64s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'ms/launch':>10s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:64s} {cnt[k]:8d} {v:10.2f} {100 * v / all_ms:6.1f}% {v / cnt[k]:10.4f}")
