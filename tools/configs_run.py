"""Full-size C2 and C5 runs through the public API (wall clock, host sampling included).

    python tools/configs_run.py [--c5-n 28] [--c5-count 2000] -> one JSON line per workload
C2: sample_permanents(EnsembleSpec("haar-u", 23, 50000, 2602)), the BASELINE config.
C5: sweep(n, "cycle" | "dft", 101) and EnsembleSpec(kind, n, count, 2602) for the five C5 kinds.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import ensembles, geodesics  # noqa: E402


def timed(fn):
    t = time.perf_counter()
    v = fn()
    return v, time.perf_counter() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5-n", type=int, default=28)
    ap.add_argument("--c5-count", type=int, default=2000)
    args = ap.parse_args()
    # warm the sampler pool and the GPU clocks
    ensembles.sample_permanents(ensembles.EnsembleSpec("haar-u", 23, 4096, 1))
    spec = ensembles.EnsembleSpec("haar-u", 23, 50000, 2602)
    v, dt = timed(lambda: ensembles.sample_permanents(spec))
    upd = spec.count * 23 * 2.0 ** 23
    print(json.dumps({"workload": "C2 haar-u n=23 x 50000", "wall_s": dt, "row_updates_per_s": upd / dt,
                      "mean_abs_perm": float(np.mean(np.abs(v)))}), flush=True)
    n = args.c5_n
    for target in ("cycle", "dft"):
        tr, dt = timed(lambda: geodesics.sweep(n, target, 101))
        print(json.dumps({"workload": f"C5 sweep {target} n={n} x 101", "wall_s": dt,
                          "row_updates_per_s": 101 * n * 2.0 ** n / dt,
                          "perm_mid": str(tr.perms[50])}), flush=True)
    for kind in ("gue", "goe", "ginibre-c", "ginibre-r", "haar-o"):
        s = ensembles.EnsembleSpec(kind, n, args.c5_count, 2602)
        v, dt = timed(lambda: ensembles.sample_permanents(s))
        print(json.dumps({"workload": f"C5 {kind} n={n} x {s.count}", "wall_s": dt,
                          "row_updates_per_s": s.count * n * 2.0 ** n / dt,
                          "mean_abs_perm": float(np.mean(np.abs(v)))}), flush=True)


if __name__ == "__main__":
    main()
