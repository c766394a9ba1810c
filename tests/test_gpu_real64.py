"""Real fp64 walks beyond n = 48 (kMaxNReal = 64): the paper's single-GPU 54 x 54
real Glynn permanent needs 54 rows of register state; the
reference engine stops at n = 40 (engine.py:25, _check_gray_dims).

A default tile at these n is 2^(m - 17) indices per lane (2^36 at n = 54): far
too long for an oracle comparison, so the tests force shorter segments with the
library's $PK_PLAN_K hook (the same kernels, only the segment length differs)
and compare whole tiles against the oracle with the S-scaled bound of
test_gpu_parity.test_large_n_tile_vs_oracle.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_2602_10141_b200 import engine, ensembles
from paper_2602_10141_b200.engine import LimitError

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.mark.parametrize("n,algo", [(49, "ryser"), (54, "glynn"), (57, "ryser"),
                                    (63, "ryser"), (64, "glynn")])
def test_real_beyond_48_tiles_vs_oracle(gpu, monkeypatch, n, algo):
    monkeypatch.setenv("PK_PLAN_K", "10")  # tiles of 32 segments of 2^10 indices
    a = np.abs(ensembles.sample_matrix("ginibre-r", n, 2602, 1)) / np.sqrt(n)
    m = n if algo == "ryser" else n - 1
    span = 8 << 15  # eight tiles
    st = int(np.random.default_rng(n).integers(0, (1 << m) // span - 1)) * span
    parts = 64
    rows = oracle.run_blocks(a, [st + i * (span // parts) for i in range(parts)],
                             [span // parts] * parts, algo)
    ref = oracle.kahan_combine(rows, False)
    s, c, ab = gpu.ryser_f64(a, algo, st, span, want_abs=True)
    assert abs((s + c) - ref) <= 8 * n * U * ab + 4 * U * abs(ref), (n, algo)
    # an unaligned range through the same kernels (ragged ends in the exact kernel);
    # the oracle walks it in 64 blocks too (one long sequential block drifts: its
    # row sums are never rebuilt, unlike the GPU's every 2^12 steps)
    st2, ln2 = st + 12345, span - 23456
    cuts = [st2 + (ln2 * i) // parts for i in range(parts + 1)]
    rows = oracle.run_blocks(a, cuts[:-1], [b - x for x, b in zip(cuts[:-1], cuts[1:])], algo)
    ref2 = oracle.kahan_combine(rows, False)
    s2, c2, ab2 = gpu.ryser_f64(a, algo, st2, ln2, want_abs=True)
    assert abs((s2 + c2) - ref2) <= 8 * n * U * ab2 + 4 * U * abs(ref2), (n, algo)


def test_real_limits(gpu):
    real = np.ones((65, 65))
    with pytest.raises(LimitError):
        engine.perm_glynn(real)
    with pytest.raises(LimitError):
        engine.perm_ryser(np.ones((64, 64)))
    with pytest.raises(LimitError):
        engine.perm_glynn(np.ones((49, 49), dtype=complex))



def _sparse_sign_matrix(n, cplx, seed):
    """Ryser test matrix for an exact signed-input check (n even, L = n / 2 "low"
    columns 0..L-1): row i has two nonzeros in {+-1} (complex: {+-1, +-i}), one in
    a low and one in a high column, each column holding two (a random cycle through
    alternately low and high columns).  Every row sum is in {0, +-1, +-i, +-2, ...}
    with |r| <= 2, so every product of the walk is an exact (Gaussian) integer."""
    rng = np.random.default_rng(seed)
    L = n // 2
    low, high = rng.permutation(L), L + rng.permutation(n - L)
    cyc = [c for pair in zip(low, high) for c in pair]  # low, high, low, high, ...
    a = np.zeros((n, n), dtype=complex if cplx else float)
    for i in range(n):
        for j in (cyc[i], cyc[(i + 1) % n]):
            a[i, j] = rng.choice([-1.0, 1.0]) * (1j if cplx and rng.random() < 0.5 else 1.0)
    return a


def _gray_inverse(g):
    b = 0
    while g:
        b ^= g
        g >>= 1
    return b


def _primes_1mod4(count):
    from paper_2602_10141_b200.modular import is_probable_prime
    out, p = [], (1 << 31) - 3
    while len(out) < count:
        if p % 4 == 1 and is_probable_prime(p):
            out.append(p)
        p -= 2
    return out


def _sqrt_minus1(p):
    c = 2
    while pow(c, (p - 1) // 2, p) != p - 1:
        c += 1
    return pow(c, (p - 1) // 4, p)


def _lift(residues, primes):
    P = 1
    for p in primes:
        P *= p
    x = 0
    for r, p in zip(residues, primes):
        q = P // p
        x += r * q * pow(q, -1, p)
    x %= P
    return x - P if x > P // 2 else x


@pytest.mark.parametrize("n,cplx", [(40, True), (44, True), (46, False), (48, False)])
def test_signed_integer_inputs_exact_at_max_sizes(gpu, monkeypatch, n, cplx):
    """A rigorous gate for SIGNED inputs at the largest n (the S-scaled tolerance of
    the max-size tests is only rigorous for nonnegative inputs).  With
    the matrices above every row sum and product of the fp64 walk is exact, so the
    production walk's only error is its compensated summation.  The range is the
    aligned block of 2^L Gray indices whose high columns are all in the subset:
    there every low column sits in two rows whose high parts h1, h2 are fixed, so the
    range sum factorises into prod over low columns of -(h1 a2 + a1 h2 + a1 a2),
    a nonzero integer (three units never cancel), reached through terms that cancel
    in sign and through row sums that cancel (h + a = 0).  The exact value comes from
    the bit-exact F_p walks of the same range (three primes p = 1 mod 4, i -> +-sqrt(-1)
    mod p separating Re and Im, CRT lift).  Gate: |(s + c) - E| <= 2u|E| + 2^-70 S."""
    from fractions import Fraction
    monkeypatch.setenv("PK_PLAN_K", "12")
    a = _sparse_sign_matrix(n, cplx, n)
    L = n // 2
    high_mask = ((1 << n) - 1) ^ ((1 << L) - 1)
    st = _gray_inverse(high_mask) & ~((1 << L) - 1)  # gray(st + t) has every high column
    span = 1 << L
    s, c, ab = gpu.ryser_f64(a, "ryser", st, span, want_abs=True)
    assert ab > 0
    primes = _primes_1mod4(3)
    re_res, im_res = [], []
    for p in primes:
        g = _sqrt_minus1(p)
        r = []
        for gg in ((g, p - g) if cplx else (0,)):
            mat = np.array([[(int(v.real) + int(v.imag) * gg) % p for v in row] for row in a],
                           dtype=np.uint64)
            r.append(gpu.ryser_modp(mat[None], [p], "ryser", st, span)[0])
        if cplx:
            inv2 = pow(2, -1, p)
            re_res.append((r[0] + r[1]) * inv2 % p)
            im_res.append((r[0] - r[1]) * inv2 * pow(g, -1, p) % p)
        else:
            re_res.append(r[0])
    exact = [_lift(re_res, primes)] + ([_lift(im_res, primes)] if cplx else [])
    got = [(complex(s).real, complex(c).real)] + \
        ([(complex(s).imag, complex(c).imag)] if cplx else [])
    for (gs, gc), E in zip(got, exact):
        err = abs(Fraction(gs) + Fraction(gc) - E)
        assert err <= 2 * Fraction(U) * abs(E) + Fraction(2) ** -70 * Fraction(ab), (n, E)
    assert any(E != 0 for E in exact)
