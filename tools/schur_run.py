"""C4 runs: exact perm(S_n) for large odd n on one B200, cross-checked on a second prime basis.

    python tools/schur_run.py 37 39 41 43 [--check 37 39]  -> gpurun_out/schur_c4.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import modular  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ns", type=int, nargs="+")
    ap.add_argument("--check", type=int, nargs="*", default=[])
    ap.add_argument("--out", default="gpurun_out/schur_c4.json")
    args = ap.parse_args()
    rows = []
    modular.schur_permanent_fast(21)  # warm-up (context, module load)
    for n in args.ns:
        t0 = time.perf_counter()
        v, b, w = modular.schur_permanent_fast(n)
        dt = time.perf_counter() - t0
        row = {"n": n, "value": str(v), "basis": list(b.primes), "residues": [x.residue for x in w],
               "wall_s": dt, "row_updates": len(b.primes) * n * 2.0 ** n,
               "prime_updates_per_s": len(b.primes) * n * 2.0 ** n / dt}
        if n in args.check:
            t0 = time.perf_counter()
            v2, b2, w2 = modular.schur_permanent_exact(n, max_bits=31)
            row["check_basis"] = list(b2.primes)
            row["check_value"] = str(v2)
            row["check_wall_s"] = time.perf_counter() - t0
            row["agree"] = v2 == v
        rows.append(row)
        print(json.dumps(row), flush=True)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
