"""Touch every kernel family once at small sizes, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck  python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
    compute-sanitizer --tool synccheck python tools/sanitize_smoke.py
    compute-sanitizer --tool initcheck python tools/sanitize_smoke.py

Families: fp64 walk (column 0 in the parameter, and batched with per-warp
slots), the fold / tree reductions, the bit-exact block kernels, F_p walks
(reduced, lazy, hybrid with narrow and wide fp64 primes, Montgomery-64), the
ragged-piece parity walker, resident jobs, and the peak / latency probes.
Results are checked loosely (the parity tests are elsewhere); the point is a
clean sanitizer report.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native as nat  # noqa: E402
from paper_2602_10141_b200 import engine, ensembles, modular  # noqa: E402


def main():
    nat.require_gpu()
    n = 18
    a = ensembles.sample_matrix("haar-u", n, 1, 0)
    r = ensembles.sample_matrix("haar-o", n, 1, 1)
    for m in (a, r):
        for algo in ("ryser", "glynn"):
            nat.ryser_f64(m, algo, 0, 1 << (n if algo == "ryser" else n - 1), 1, want_abs=True)
            nat.ryser_f64(m, algo, 12345, 70000, 1)  # ragged head / tail pieces
    nat.ryser_f64_blocks(a, "ryser", [0, 777], [1000, 3000])
    engine.perm_batch(np.stack([ensembles.sample_matrix("gue", 12, 2, i) for i in range(9)]))
    engine.perm_batch(np.stack([ensembles.sample_matrix("goe", 12, 2, i) for i in range(9)]),
                      method="glynn")
    n = 20
    ps = (modular.prime_pool(n, "reduced", 2) + modular.prime_pool(n, "lazy", 3)
          + modular.prime_pool(n, "fp64", 1) + modular.prime_pool(n, "fp64w", 1)
          + list(modular.find_primes(n, max_bits=59).primes[:1]) + [15, 4])
    mats = np.stack([modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n))
                     if p > 16 else np.full((n, n), 3 % p, dtype=np.uint64) for p in ps])
    for algo in ("ryser", "glynn"):
        nat.ryser_modp(mats, ps, algo, 0, 1 << (n - 1))
        nat.ryser_modp(mats, ps, algo, 999, 40000)
    job = nat.Job.modp(mats[:-2], ps[:-2], "ryser", 0, 1 << n)
    job.run(2)
    job.close()
    job = nat.Job.f64(a[:16, :16].copy(), "ryser", 0, 1 << 16)
    job.run(2, 1 << 20)
    job.close()
    print("sanitize smoke: every kernel family ran")


if __name__ == "__main__":
    main()
