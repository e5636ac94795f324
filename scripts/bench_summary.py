"""Print the headline fields of a bench.py JSON line (debug helper)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("ms/solve %.1f  value %.3e  relax0 %.3f ms  frac %.3f  e2e %s" % (
    d["ms_per_step"], d["value"], d["roofline"]["mean_launch_ms"], d["roofline"]["frac"],
    d.get("e2e", {}).get("value")))
print({k: round(v["ms_per_solve"], 1) for k, v in d["kernels"].items() if isinstance(v, dict)})
