"""Permanent engines over the B200 Gray-code walk.

Public surface and error behaviour follow the reference engine
(reference pkg/src/permkit/engine.py:24-320): ``permanent``, ``perm_ryser``,
``perm_glynn``, ``perm_blocked``, ``perm_naive``, ``perm_abs_entrywise``,
``KahanAccumulator`` and ``LimitError``, with the same exceptions, messages and
return types (complex for COMPLEX, float for REAL, int for INTEGER and F_p,
Fraction for RATIONAL).

What changes is where the walk runs.  The reference cuts [0, 2^m) into a plan
of 64 x threads blocks and evaluates each block in a numba thread
(engine.py:213-245).  Here one call covers the whole range on the GPU:

* COMPLEX / REAL -> ``pk_ryser_f64``: aligned segments per lane, Neumaier per
  lane, deterministic tree over lanes / tiles / devices.
* PrimeField(p)  -> ``pk_ryser_modp`` (exact).
* INTEGER        -> several word-size primes in ONE pass of ``pk_ryser_modp``,
  then a symmetric CRT lift; the prime set covers 2 * prod_i ||a_i||_1 + 1, a
  bound on |perm| (the reference walks Python big ints, engine.py:130-192).
* RATIONAL       -> rows scaled to integers by their denominators' lcm.

``threads`` is accepted for signature compatibility and ignored: the GPU
chooses its own decomposition.  ``devices`` (or $PERMKIT_GPU_DEVICES) splits a
walk over that many GPUs; for power-of-two device counts the result is
bit-identical to one device.  There is no CPU fallback: without the library or
a device every call raises ``GpuUnavailableError``.
"""

from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

from . import _native
from .domains import COMPLEX, INTEGER, RATIONAL, REAL, PrimeField, ScalarDomain, infer_domain
from .gray import GLYNN, RYSER, BlockPlan, iteration_exponent

NAIVE_MAX_N = 11
GRAY_MAX_N = 48   # reference: 40 (engine.py:25); lifted to the GPU kernels' range
# real fp64 walks: 64 rows of state fit the register file (the paper's 54 x 54
# real Glynn permanent); Ryser's 2^64 range of n = 64 does not
# fit a uint64 length, so Ryser stops at 63
REAL_MAX_N = {RYSER: 63, GLYNN: 64}
ABS_MAX_N = 25


class LimitError(Exception):
    """A documented capability limit was exceeded (CLI exit code 3)."""


class KahanAccumulator:
    """Neumaier-compensated running sum, one error-free transform per component.

    Same semantics as the reference accumulator (engine.py:33-73): ``add``
    takes a complex or real value, ``value`` is sum + compensation.
    """

    __slots__ = ("_parts", "_cplx")

    def __init__(self, complex_valued: bool = False):
        self._parts = [0.0, 0.0, 0.0, 0.0]  # sum_re, comp_re, sum_im, comp_im
        self._cplx = complex_valued

    @staticmethod
    def _two(s, c, v):
        t = s + v
        big, small = (s, v) if abs(s) >= abs(v) else (v, s)
        return t, c + ((big - t) + small)

    def add(self, value):
        z = complex(value)
        p = self._parts
        p[0], p[1] = self._two(p[0], p[1], z.real)
        if self._cplx:
            p[2], p[3] = self._two(p[2], p[3], z.imag)

    @property
    def sum(self):
        p = self._parts
        return complex(p[0], p[2]) if self._cplx else p[0]

    @property
    def compensation(self):
        p = self._parts
        return complex(p[1], p[3]) if self._cplx else p[1]

    @property
    def value(self):
        p = self._parts
        if self._cplx:
            return complex(p[0] + p[1], p[2] + p[3])
        return p[0] + p[1]


# ---------------------------------------------------------------------------
# input handling (reference engine.py:76-112)

def _normalize(a, domain):
    if domain is None:
        a = np.asarray(a)
        domain = infer_domain(a)
    if isinstance(a, np.ndarray):
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("matrix must be square")
        n = a.shape[0]
        rows = None
    else:
        rows = [list(r) for r in a]
        n = len(rows)
        if any(len(r) != n for r in rows):
            raise ValueError("matrix must be square")
    if n == 0:
        raise ValueError("empty matrix")
    if domain is COMPLEX or domain is REAL:
        src = a if rows is None else np.array(rows, dtype=object)
        dt = np.complex128 if domain is COMPLEX else np.float64
        return np.ascontiguousarray(src, dtype=dt), domain, n
    src = a if rows is None else rows
    conv = (lambda v: int(v) % domain.p) if isinstance(domain, PrimeField) else domain.coerce
    out = np.empty((n, n), dtype=object)
    for i in range(n):
        for j in range(n):
            out[i, j] = conv(src[i][j])
    return out, domain, n


def _check_gray_dims(n, domain=None, algorithm=None):
    if domain is REAL and algorithm in REAL_MAX_N and n > GRAY_MAX_N:
        if n > REAL_MAX_N[algorithm]:
            raise LimitError(f"dimension {n} exceeds the n <= {REAL_MAX_N[algorithm]} range "
                             f"of real {algorithm}")
        return
    if n > GRAY_MAX_N:
        raise LimitError(f"dimension {n} exceeds the n <= {GRAY_MAX_N} range")


def _validate_plan(plan: BlockPlan, n: int):
    if plan.n != n:
        raise ValueError("plan dimension does not match matrix")
    if plan.total != (1 << iteration_exponent(n, plan.algorithm)):
        raise ValueError("plan does not cover the iteration range")
    pos = 0
    for blk in plan.blocks:
        if blk.start != pos or blk.length < 0:
            raise ValueError("plan blocks must be contiguous and ordered")
        pos += blk.length


def _devices(devices):
    return int(devices) if devices else _native.default_devices()


# ---------------------------------------------------------------------------
# naive oracle API (host; n <= 11)

def perm_naive(a, domain: ScalarDomain | None = None):
    """Permanent as the sum over all n! permutations (reference engine.py:115-127)."""
    a, domain, n = _normalize(a, domain)
    if n > NAIVE_MAX_N:
        raise LimitError("oracle dimension exceeded")
    acc = domain.zero()
    for sigma in itertools.permutations(range(n)):
        term = domain.one()
        for i, j in enumerate(sigma):
            term = domain.mul(term, a[i, j])
        acc = domain.add(acc, term)
    return acc


# ---------------------------------------------------------------------------
# exact integers through F_p walks + CRT

def _is_probable_prime(n: int) -> bool:
    from .modular import is_probable_prime
    return is_probable_prime(n)


def integer_crt_primes(n: int, bound: int) -> list:
    """Odd primes p with n (p - 1) < 2^31 (the lazy Montgomery kernel) whose
    product exceeds 2 * bound + 1, largest first."""
    top = ((1 << 31) - 1) // n + 1
    primes, prod = [], 1
    p = top if top % 2 else top - 1
    while prod <= 2 * bound + 1:
        if p < 3:
            raise ValueError("prime supply exhausted for the CRT bound")
        if _is_probable_prime(p):
            primes.append(p)
            prod *= p
        p -= 2
    return primes


def _crt_lift(residues, primes) -> int:
    prod = math.prod(primes)
    x = 0
    for r, p in zip(residues, primes):
        m = prod // p
        x += r * m * pow(m, -1, p)
    x %= prod
    return x - prod if x > prod // 2 else x


def _exact_int_perm(rows, n: int, algorithm: str, devices) -> int:
    # The exact value does not depend on the expansion, so the walk is always
    # Glynn's: 2^(n-1) sign vectors instead of Ryser's 2^n subsets, same cost
    # per step (the CRT primes are odd, so 2^(n-1) is invertible).
    algorithm = GLYNN
    bound = 1
    for r in rows:
        bound *= sum(abs(int(v)) for v in r)
    if bound == 0:
        return 0
    primes = integer_crt_primes(n, bound)
    res = np.array([[[int(v) % p for v in r] for r in rows] for p in primes], dtype=np.uint64)
    m = iteration_exponent(n, algorithm)
    raw = _native.ryser_modp(res, primes, algorithm, 0, 1 << m, _devices(devices))
    if algorithm == GLYNN:
        raw = [x * pow(pow(2, n - 1, p), -1, p) % p for x, p in zip(raw, primes)]
    return _crt_lift(raw, primes)


def _exact_perm(a, domain, n, algorithm, devices):
    if domain is INTEGER:
        return _exact_int_perm([[int(a[i, j]) for j in range(n)] for i in range(n)], n,
                               algorithm, devices)
    if domain is RATIONAL:
        scale = 1
        rows = []
        for i in range(n):
            fr = [Fraction(a[i, j]) for j in range(n)]
            d = math.lcm(*[f.denominator for f in fr])
            scale *= d
            rows.append([int(f * d) for f in fr])
        return Fraction(_exact_int_perm(rows, n, algorithm, devices), scale)
    raise TypeError(f"no GPU path for domain {domain!r}")


# ---------------------------------------------------------------------------
# GPU evaluation of a whole range / a plan

def _float_result(value, domain, n, algorithm):
    if algorithm == GLYNN:
        value = value * (2.0 ** (1 - n))
    if domain is REAL:
        return float(value.real) if isinstance(value, complex) else float(value)
    return value


def _run_full(a, domain, n, algorithm, devices):
    m = iteration_exponent(n, algorithm)
    if domain is COMPLEX or domain is REAL:
        s, c, _ = _native.ryser_f64(a, algorithm, 0, 1 << m, _devices(devices))
        return _float_result(s + c, domain, n, algorithm)
    if isinstance(domain, PrimeField):
        p = domain.p
        au = np.array([[int(v) for v in row] for row in a], dtype=np.uint64)
        r = _native.ryser_modp(au[None], [p], algorithm, 0, 1 << m, _devices(devices))[0]
        return domain.div_pow2(r, n - 1) if algorithm == GLYNN else r
    return _exact_perm(a, domain, n, algorithm, devices)


def _run_plan(a, domain, plan, devices):
    """Evaluate a caller's plan block by block and combine in block order.

    fp64: each block is one GPU range walk returning a compensated pair; the
    pairs are folded with KahanAccumulator add(s); add(c) exactly as the
    reference does (engine.py:240-245), so the result depends on the plan but
    never on the worker count.  Exact domains are plan-independent.
    """
    n = a.shape[0]
    _validate_plan(plan, n)
    algorithm = plan.algorithm
    if domain is COMPLEX or domain is REAL:
        # one C-ABI call for the whole plan (pk_ryser_f64_plan): every block's
        # pair is the one a single-range call on it returns; then the
        # reference's ordered KahanAccumulator combine (pk_kahan_fold)
        parts, _ = _native.ryser_f64_plan(a, algorithm, [b.start for b in plan.blocks],
                                          [b.length for b in plan.blocks], _devices(devices))
        s, c = _native.kahan_fold(parts, domain is COMPLEX)
        return _float_result(s + c, domain, n, algorithm)
    return _run_full(a, domain, n, algorithm, devices)


# ---------------------------------------------------------------------------
# public API

def perm_blocked(a, plan: BlockPlan, worker_count: int = 1,
                 domain: ScalarDomain | None = None, devices: int | None = None):
    """Permanent via a block plan; bit-identical for any worker_count."""
    a, domain, n = _normalize(a, domain)
    _check_gray_dims(n, domain, plan.algorithm)
    if isinstance(domain, PrimeField) and plan.algorithm == GLYNN and domain.p == 2:
        raise ValueError("division by two unavailable in GF(2)")
    return _run_plan(a, domain, plan, devices)


def perm_ryser(a, domain: ScalarDomain | None = None, threads: int = 1,
               devices: int | None = None):
    """Ryser's inclusion-exclusion permanent in Gray-code order (GPU)."""
    a, domain, n = _normalize(a, domain)
    _check_gray_dims(n, domain, RYSER)
    return _run_full(a, domain, n, RYSER, devices)


def perm_glynn(a, domain: ScalarDomain | None = None, threads: int = 1,
               devices: int | None = None):
    """Glynn's 2^(n-1)-term expansion in Gray-code order (GPU)."""
    a, domain, n = _normalize(a, domain)
    _check_gray_dims(n, domain, GLYNN)
    if isinstance(domain, PrimeField) and domain.p == 2:
        raise ValueError("division by two unavailable in GF(2)")
    return _run_full(a, domain, n, GLYNN, devices)


def permanent(a, method: str = "ryser", domain: ScalarDomain | None = None,
              threads: int = 1, devices: int | None = None):
    """Dispatch by method name ("naive", "ryser", "glynn")."""
    if method == "naive":
        return perm_naive(a, domain)
    if method == RYSER:
        return perm_ryser(a, domain, threads, devices)
    if method == GLYNN:
        return perm_glynn(a, domain, threads, devices)
    raise ValueError(f"unknown method {method!r}")


def perm_abs_entrywise(a, threads: int = 1, devices: int | None = None) -> float:
    """Permanent of the entrywise absolute-value matrix."""
    a = np.asarray(a)
    n = a.shape[0]
    if n > ABS_MAX_N:
        raise LimitError(f"dimension {n} exceeds the n <= {ABS_MAX_N} range")
    mags = np.ascontiguousarray(np.abs(a).astype(np.float64))
    return float(perm_ryser(mags, REAL, threads=threads, devices=devices))


def perm_batch(mats, method: str = "ryser", devices: int | None = None,
               want_abs: bool = False):
    """Permanents of a stack of fp64 matrices [B, n, n] in one GPU pass.

    Returns complex128 [B] for complex input and float64 [B] for real input
    (plus the per-matrix sum |term| bound when ``want_abs``).  This is the
    batched form behind ``sample_permanents`` and ``sweep``.
    """
    mats = np.asarray(mats)
    if mats.ndim != 3 or mats.shape[1] != mats.shape[2]:
        raise ValueError("expected a stack of square matrices [B, n, n]")
    B, n = mats.shape[0], mats.shape[1]
    if n == 0:
        raise ValueError("empty matrix")
    if method == "naive":
        vals = np.array([perm_naive(m) for m in mats])
        return (vals, None) if want_abs else vals
    _check_gray_dims(n, COMPLEX if np.iscomplexobj(mats) else REAL, method)
    if method not in (RYSER, GLYNN):
        raise ValueError(f"unknown method {method!r}")
    cplx = np.iscomplexobj(mats)
    if B == 0:
        out = np.zeros(0, dtype=np.complex128 if cplx else np.float64)
        return (out, np.zeros(0)) if want_abs else out
    raw, ab = _native.ryser_f64_batch(mats, method, _devices(devices), want_abs)
    if cplx:
        vals = (raw[:, 0] + raw[:, 2]) + 1j * (raw[:, 1] + raw[:, 3])
    else:
        vals = raw[:, 0] + raw[:, 2]
    if method == GLYNN:
        vals = vals * (2.0 ** (1 - n))
    return (vals, ab) if want_abs else vals
