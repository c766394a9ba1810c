"""Rate of the exact per-block kernel (pk_ryser_f64_blocks, csrc/pk_block.cuh).

    PERMKIT_GPU_LIB=<lib.so> python tools/block_rate.py   -> one JSON line per case

The block kernel is the reference-exact walk (kernels.py:33-226 arithmetic); it
serves the parity API, perm_blocked plans and ragged pieces of unaligned ranges.
Each case walks 148 * 128 blocks of L steps on one matrix; the line carries the
rate (block steps/s) and a hash of the returned bits, so two libraries can be
compared for both speed and bit identity.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native  # noqa: E402

CASES = [(True, "ryser", 20), (True, "ryser", 32), (True, "glynn", 32), (False, "ryser", 32),
         (True, "ryser", 48), (False, "glynn", 48), (False, "glynn", 64)]


def main():
    rng = np.random.default_rng(7)
    nb = 148 * 128
    for cplx, algo, n in CASES:
        a = rng.standard_normal((n, n)) / np.sqrt(n)
        if cplx:
            a = a + 1j * rng.standard_normal((n, n)) / np.sqrt(n)
        m = n if algo == "ryser" else n - 1
        L = 4096 if n <= 32 else 1024
        starts = (np.arange(nb, dtype=np.uint64) * np.uint64(L * 3 + 1)) % np.uint64((1 << m) - L)
        lens = np.full(nb, L, dtype=np.uint64)
        _native.ryser_f64_blocks(a, algo, starts[:64], lens[:64])  # warm
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            out = _native.ryser_f64_blocks(a, algo, starts, lens)
            best = min(best, time.perf_counter() - t0)
        print(json.dumps({"cplx": cplx, "algo": algo, "n": n, "blocks": nb, "len": L,
                          "s": round(best, 5), "block_steps_per_s": nb * L / best,
                          "bits": hashlib.sha1(np.ascontiguousarray(out).tobytes()).hexdigest()[:16]}),
              flush=True)


if __name__ == "__main__":
    main()
