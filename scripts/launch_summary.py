"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel
and grid shape (for the level kernels the grid identifies the level)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0].replace("unnamed>::", "").replace("void ", "")
    key = f"{name} grid{r[8]}" if ("k_relax_tma" in name or "k_materialize" in name) else name
    tot[key] += float(r[-1]) * 1e-6
    cnt[key] += 1
all_ms = sum(tot.values())
print(f"{len(rows)} launches, {all_ms:.1f} ms total (serialised, cold-cache ncu timings)")
print(f"{'kernel':64s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'ms/launch':>10s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:64s} {cnt[k]:8d} {v:10.2f} {100 * v / all_ms:6.1f}% {v / cnt[k]:10.4f}")
