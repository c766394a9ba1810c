"""First-contact GPU probe: pipe peaks, F_p / fp64 sanity, and first timings.

Run on the B200 box:  python tools/gpu_probe.py  (writes gpurun_out/probe.json)
Self-contained (numpy + the built library); no reference import.
"""
import itertools
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native as nat  # noqa: E402


def is_prime(n):
    if n < 2:
        return False
    for q in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for w in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(w, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def primes_1modn(n, below, count):
    out, k = [], (below - 2) // n
    while len(out) < count:
        p = k * n + 1
        if p > 2 and is_prime(p):
            out.append(p)
        k -= 1
    return out


def prim_root(p, n):
    if n == 1:
        return 1
    fac, m, d = set(), n, 2
    while d * d <= m:
        while m % d == 0:
            fac.add(d)
            m //= d
        d += 1
    if m > 1:
        fac.add(m)
    e = (p - 1) // n
    for c in range(2, p):
        g = pow(c, e, p)
        if g != 1 and all(pow(g, n // q, p) != 1 for q in fac):
            return g


def schur_res(n, p):
    g = prim_root(p, n)
    pw = [pow(g, k, p) for k in range(n)]
    return np.array([[pw[(j * k) % n] for k in range(n)] for j in range(n)], dtype=np.uint64)


def crt(res, ps):
    P = math.prod(ps)
    x = sum(r * (P // p) * pow(P // p, -1, p) for r, p in zip(res, ps)) % P
    return x - P if x > P // 2 else x


def perm_naive(a):
    n = a.shape[0]
    return sum(np.prod([a[i, s[i]] for i in range(n)]) for s in itertools.permutations(range(n)))


def main():
    rep = {}
    print("devices", nat.device_count(), flush=True)
    t = time.time()
    rep["peaks"] = nat.measure_peaks(0)
    print(json.dumps(rep["peaks"], indent=1), "in", time.time() - t, flush=True)

    known = {13: 175747, 15: 30375, 17: 25219857, 19: 142901109, 21: 4548104883,
             23: -31152650265, 25: -5198937484375}
    rep["schur"] = {}
    for n, want in known.items():
        for mode, below in (("lazy", (1 << 31) // n), ("reduced", 1 << 31)):
            ps = primes_1modn(n, below, 4)
            mats = np.stack([schur_res(n, p) for p in ps])
            t = time.time()
            r = nat.ryser_modp(mats, ps, "ryser", 0, 1 << n)
            dt = time.time() - t
            # ryser_modp returns the signed walk sum = perm mod p
            got = crt(r, ps)
            ok = got == want
            rep["schur"][f"{n}_{mode}"] = {"ok": ok, "got": got, "s": dt}
            print("schur", n, mode, ok, got, want, f"{dt:.3f}s", flush=True)
    # glynn mod p: raw sum * 2^(1-n)
    n = 15
    ps = primes_1modn(n, (1 << 31) // n, 2)
    mats = np.stack([schur_res(n, p) for p in ps])
    r = nat.ryser_modp(mats, ps, "glynn", 0, 1 << (n - 1))
    r = [x * pow(pow(2, n - 1, p), -1, p) % p for x, p in zip(r, ps)]
    print("glynn modp n=15", crt(r, ps), "want", known[15], flush=True)

    rng = np.random.default_rng(1)
    rep["f64"] = {}
    for n in (3, 5, 8, 9):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        want = perm_naive(a)
        s, c, _ = nat.ryser_f64(a, "ryser", 0, 1 << n)
        got = s + c
        g2s, g2c, _ = nat.ryser_f64(a, "glynn", 0, 1 << (n - 1))
        got2 = (g2s + g2c) * 2.0 ** (1 - n)
        print("f64 n", n, got, want, abs(got - want) / abs(want), abs(got2 - want) / abs(want), flush=True)
        rep["f64"][n] = [abs(got - want) / abs(want), abs(got2 - want) / abs(want)]
    for n in (14, 20, 24):
        for cplx in (True, False):
            a = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
            a = a / math.sqrt(n)
            s, c, ab = nat.ryser_f64(a, "ryser", 0, 1 << n, want_abs=True)
            blk = nat.ryser_f64_blocks(a, "ryser", [0], [1 << n])[0]
            ex = complex(blk[0], blk[1]) + complex(blk[2], blk[3])
            gs, gc, _ = nat.ryser_f64(a, "glynn", 0, 1 << (n - 1))
            gl = (gs + gc) * 2.0 ** (1 - n)
            err = abs((s + c) - ex)
            print("f64", n, cplx, "prod vs exact-block", err, "tol", 2 * n * 2 ** -53 * ab,
                  "glynn diff", abs(gl - ex), flush=True)
            rep["f64"][f"{n}_{cplx}"] = [err, 2 * n * 2 ** -53 * ab]
    # batch
    B, n = 64, 16
    mats = (rng.standard_normal((B, n, n)) + 1j * rng.standard_normal((B, n, n))) / 4
    out, _ = nat.ryser_f64_batch(mats, "ryser")
    singles = [sum(nat.ryser_f64(m, "ryser", 0, 1 << n)[:2]) for m in mats[:4]]
    print("batch", [complex(o[0], o[1]) + complex(o[2], o[3]) for o in out[:4]], singles, flush=True)

    # timings
    q, _ = np.linalg.qr(rng.standard_normal((32, 32)) + 1j * rng.standard_normal((32, 32)))
    for n, cplx in ((32, True), (32, False), (28, True)):
        a = q[:n, :n] if cplx else q[:n, :n].real.copy()
        job = nat.Job.f64(a, "ryser", 0, 1 << n)
        job.run(1)
        tot, walk, res = job.run(3)
        ups = 3 * n * 2.0 ** n / (walk / 1e3)
        print("f64 job", n, cplx, job.info(), f"walk {walk/3:.2f} ms/run", f"{ups:.3e} upd/s",
              flush=True)
        rep[f"time_f64_{n}_{cplx}"] = {"ms": walk / 3, "ups": ups, **job.info()}
        job.close()
    for n in (32, 36):
        for mode, below in (("lazy", (1 << 31) // n), ("reduced", 1 << 31)):
            ps = primes_1modn(n, below, 4)
            mats = np.stack([schur_res(n, p) for p in ps])
            job = nat.Job.modp(mats, ps, "ryser", 0, 1 << n)
            job.run(1)
            tot, walk, res = job.run(2 if n == 32 else 1)
            it = 2 if n == 32 else 1
            ups = it * 4 * n * 2.0 ** n / (walk / 1e3)
            print("modp job", n, mode, job.info(), f"walk {walk/it:.2f} ms/run", f"{ups:.3e} upd/s",
                  "res", res, flush=True)
            rep[f"time_modp_{n}_{mode}"] = {"ms": walk / it, "ups": ups, "res": res, **job.info()}
            job.close()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/probe.json", "w") as f:
        json.dump(rep, f, indent=1, default=str)


if __name__ == "__main__":
    main()
