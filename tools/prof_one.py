"""Run one resident walk for profiling:
    python tools/prof_one.py {f64c|f64r|modp|modpr|red<P>|lazy<P>|hyb|basis|wide|batch|batchr} N [iters] [range_bits]
range_bits (default n): walk only the aligned range [0, 2^range_bits) (per-step cost is
start-independent), e.g. to keep an ncu replay of an n = 43 walk short."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native as nat  # noqa: E402
from tools.gpu_probe import primes_1modn, schur_res  # noqa: E402

kind, n = sys.argv[1], int(sys.argv[2])
if kind.startswith("batch"):
    import time
    from paper_2602_10141_b200 import ensembles, perm_batch
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
    kk = "haar-u" if kind == "batch" else "haar-o"
    mats = ensembles.sample_batch(ensembles.EnsembleSpec(kk, n, B, 2602), 0, B)
    perm_batch(mats[:64])
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    for _ in range(reps):  # reps > 1: first-call vs steady state
        t = time.perf_counter()
        perm_batch(mats)
        dt = time.perf_counter() - t
        print(kind, n, B, f"{dt * 1e3:.1f} ms", f"{B * n * 2.0 ** n / dt:.3e} upd/s (incl. H2D/D2H)",
              flush=True)
    sys.exit(0)
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 1
span = 1 << (int(sys.argv[4]) if len(sys.argv) > 4 else n)
rng = np.random.default_rng(3)
if kind.startswith("f64"):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    a = q if kind == "f64c" else q.real.copy()
    job = nat.Job.f64(a, "ryser", 0, span)
elif kind[:3] == "red" or kind[:4] == "lazy":  # e.g. red3, lazy4: one launch group
    from paper_2602_10141_b200 import modular
    P = int(kind[-1])
    ps = modular.prime_pool(n, "reduced" if kind[:3] == "red" else "lazy", P)
    job = nat.Job.modp(np.stack([schur_res(n, p) for p in ps]), ps, "ryser", 0, span)
elif kind in ("basis", "wide"):
    from paper_2602_10141_b200 import modular
    ps = (list(modular.gpu_prime_basis(n).primes) if kind == "basis"
          else list(modular.find_primes(n, max_bits=59).primes[:1]))
    job = nat.Job.modp(np.stack([schur_res(n, p) for p in ps]), ps, "ryser", 0, span)
elif kind == "hyb":
    from paper_2602_10141_b200 import modular
    ps = modular.prime_pool(n, "lazy", 2) + modular.prime_pool(n, "fp64", 2)  # two hybrid pairs
    job = nat.Job.modp(np.stack([schur_res(n, p) for p in ps]), ps, "ryser", 0, span)
else:
    below = (1 << 31) // n if kind == "modp" else (1 << 31)
    ps = primes_1modn(n, below, 4)
    job = nat.Job.modp(np.stack([schur_res(n, p) for p in ps]), ps, "ryser", 0, span)
tot, walk, res = job.run(iters)
print(kind, n, job.info(), f"walk {walk / iters:.3f} ms", f"{iters * n * float(span) * (len(ps) if kind.startswith(('modp', 'hyb', 'basis', 'wide', 'red', 'lazy')) else 1) / (walk / 1e3):.3e} upd/s")
