"""Per-launch-group F_p walk rates on one B200, for the CRT basis cost model.

    python tools/modp_rates.py 32 36 40 43 [--bits 36] [--only wide1 wide2]  -> gpurun_out/modp_rates.json

For each n it times one resident walk over an aligned Gray range of 2^bits indices
(per-step cost is start-independent) for every launch-group shape the C ABI forms:
  red<P>   P reduced 31-bit Montgomery primes   (n (p - 1) >= 2^31)
  lazy<P>  P lazy Montgomery primes             (n (p - 1) < 2^31, not fp64-eligible)
  hyb11    one lazy Montgomery prime + one fp64 prime (walk_hybrid_kernel<n, 1, 1, false>)
  hybw11   one lazy Montgomery prime + one wide fp64 prime (walk_hybrid_kernel<n, 1, 1, true>)
  wide<P>  P 59-bit primes, Montgomery-64 (walk_modp64_kernel<n, P>)
and reports prime-row-updates/s and CRT bits/s (sum of log2 p per second).
"""
import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native as nat  # noqa: E402
from paper_2602_10141_b200 import modular  # noqa: E402
from tools.gpu_probe import schur_res  # noqa: E402


def primes_desc(n, below, count, accept):
    out, k = [], (below - 2) // n
    while len(out) < count and k >= 1:
        p = k * n + 1
        if accept(p) and modular.is_probable_prime(p):
            out.append(p)
        k -= 1
    return out


def rate(n, primes, bits, iters):
    res = np.stack([schur_res(n, p) for p in primes])
    job = nat.Job.modp(res, primes, "ryser", 0, 1 << bits)
    job.run(1)  # warm-up
    _, walk, _ = job.run(iters)
    info = job.info()
    job.close()
    upd = n * 2.0 ** bits * len(primes)
    s = walk / iters / 1e3
    return {"primes": primes, "ms": walk / iters, "prime_upd_per_s": upd / s,
            "bits_per_s": sum(math.log2(p) for p in primes) * n * 2.0 ** bits / s,
            "launches": info["launches"], "regs": info["regs"],
            "ctas_per_sm": info["ctas_per_sm"], "local_bytes": info["local_bytes"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ns", type=int, nargs="+")
    ap.add_argument("--bits", type=int, default=36)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/modp_rates.json")
    ap.add_argument("--only", nargs="*", default=None)
    args = ap.parse_args()
    rows = []
    for n in args.ns:
        bits = min(n, args.bits)
        pmax = 4 if n <= 36 else 3
        red = primes_desc(n, 1 << 31, pmax, lambda p: n * (p - 1) >= (1 << 31))
        lazy = primes_desc(n, (1 << 31) // n, pmax,
                           lambda p: n * (p - 1) < (1 << 31) and not modular.fp64_prime_ok(p, n))
        fp = primes_desc(n, 1 << 26, 1, lambda p: modular.fp64_prime_ok(p, n))
        shapes = {f"red{P}": red[:P] for P in range(1, pmax + 1)}
        shapes.update({f"lazy{P}": lazy[:P] for P in range(1, pmax + 1)})
        if n >= 17:
            shapes["hyb11"] = [lazy[0], fp[0]]
            shapes["hybw11"] = [lazy[0], modular.prime_pool(n, "fp64w", 1)[0]]
        wide = primes_desc(n, 1 << 59, 2, lambda p: True)  # reference default 59-bit basis
        shapes["wide1"] = wide[:1]
        if n <= 36:
            shapes["wide2"] = wide[:2]
        for name, ps in shapes.items():
            if args.only and name not in args.only:
                continue
            r = rate(n, ps, bits, args.iters)
            r.update({"n": n, "shape": name, "range_bits": bits})
            rows.append(r)
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) and v < 1e6 else v)
                              for k, v in r.items()}), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
