"""Hot SASS listing from `ncu -i rep --page source --csv --print-source sass`:
per-instruction executed counts, opcode histogram weighted by execution."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iE, iSm = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[iE].isdigit()]
tot = sum(int(r[iE]) for r in body)
hist = collections.Counter()
for r in body:
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    hist[o.split(".")[0]] += int(r[iE])
print("total warp instructions", tot)
for o, c in hist.most_common(30):
    print(f"  {o:12s} {c:14d} {100 * c / tot:5.1f}%")
if len(sys.argv) > 2:
    thr = float(sys.argv[2])
    mx = max(int(r[iE]) for r in body)
    for r in body:
        if int(r[iE]) >= thr * mx:
            print(r[iA][-5:], f"{int(r[iE]):12d} {r[iSm]:>6s}", r[iS].strip())
