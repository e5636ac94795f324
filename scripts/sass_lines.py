"""Join an ncu SASS source page (csv) with nvdisasm -g line info: executed
warp instructions and stall samples per source line.
usage: sass_lines.py <ncu-rep> <cubin> <function-substring>"""
import csv, re, subprocess, sys, collections

rep, cubin, fsub = sys.argv[1:4]
page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(page))
h = r[1]
rows = r[2:]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
# find the function section
start = None
for i, l in enumerate(dis):
    if l.startswith(".text.") and fsub in l:
        start = i
        break
lines = {}
cur = None
for l in dis[start + 1:]:
    if l.startswith(".text.") or l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if "inlined at" not in l:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        lines[int(m.group(1), 16)] = (cur, m.group(2))
base = int(rows[0][0], 16)
ex = collections.Counter()
st = collections.Counter()
for x in rows:
    off = int(x[0], 16) - base
    key = lines.get(off, (None, ""))[0]
    ex[key] += int(x[iE] or 0)
    st[key] += int(x[iW] or 0)
tot_e = sum(ex.values())
tot_s = sum(st.values())
print("total warp instr", tot_e, "stall samples", tot_s)
for k, v in sorted(ex.items(), key=lambda kv: -kv[1])[:40]:
    print(f"{str(k):40s} instr {v:12d} ({100*v/tot_e:5.1f}%)  stalls {100*st[k]/max(tot_s,1):5.1f}%")
