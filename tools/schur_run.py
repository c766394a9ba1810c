"""C4 runs: exact perm(S_n) for large odd n on one B200, cross-checked on a second prime
basis (31-bit, Ryser expansion: an independent walk).

    python tools/schur_run.py 37 39 41 43 [--check 37 39] [--method glynn|ryser]
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
    ap.add_argument("--method", default="glynn", choices=["glynn", "ryser"])
    args = ap.parse_args()
    rows = []
    modular.schur_permanent_fast(21)  # warm-up (context, module load)
    for n in args.ns:
        t0 = time.perf_counter()
        v, b, w = modular.schur_permanent_fast(n, method=args.method)
        dt = time.perf_counter() - t0
        upd = len(b.primes) * n * 2.0 ** (n - 1 if args.method == "glynn" else n)
        row = {"n": n, "value": str(v), "basis": list(b.primes), "residues": [x.residue for x in w],
               "expansion": args.method, "wall_s": dt, "row_updates": upd,
               "prime_updates_per_s": upd / dt}
        if n in args.check:
            t0 = time.perf_counter()
            v2, b2, w2 = modular.schur_permanent_exact(n, max_bits=31, method="ryser")
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
