"""Device problem builders against the reference's host
builders (oracle/_ref, ref_problem_fields: serial std::function / libm per
node) on the same box.  One JSON line per builder: device wall time at n
(table on the host + device fill, synchronised), reference time at n_cpu."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_07206_b200 as S  # noqa: E402
from oracle import oracle as O  # noqa: E402  (reference timing only)


def wall(fn, reps=3):
    fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return float(np.median(t))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n_cpu = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    g3 = S.make_grid(3, n)
    cases = {
        "poisson3d_problem": (lambda: S.poisson3d_source(g3), "poisson3d"),
        "capacitor_problem sigma": (lambda: S.capacitor_sigma(g3, "high"), "capacitor_high"),
        "trifoil_problem (3 sources)": (lambda: S.trifoil_sources(g3, 0.14), "trifoil_x"),
    }
    for name, (fn, ref) in cases.items():
        sec = wall(fn)
        line = {"builder": name, "n": n, "nodes": g3.total, "device_s": sec, "device_nodes_per_s": g3.total / sec}
        if O.ref_lib() is not None:
            t0 = time.perf_counter()
            O.ref_problem(ref, n_cpu)
            rs = time.perf_counter() - t0
            gc = O.make_grid(3, n_cpu)
            line.update({"ref_n": n_cpu, "ref_s": rs, "ref_nodes_per_s": gc.total / rs, "ref_kind": "reference (serial)"})
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
