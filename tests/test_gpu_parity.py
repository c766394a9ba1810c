"""GPU parity: the sm_100a kernels (through the C ABI) against the reference.

Gates:
  * F_p residues and CRT integers: bit-exact.
  * fp64, parity kernel (exact=True): bit-identical (sum, comp) per block.
  * fp64, production kernel: |gpu - exact| <= 2 n u S + 4 u |exact|, where
    u = 2^-53, S = sum over terms of |re t| + |im t| (emitted by the kernel)
    and `exact` is the big-integer block sum (tests/exact_walk.py).  Against
    the reference (which drifts along its sequential walk) the gate is
    8 n u S.  A flat relative tolerance is not achievable for Haar inputs
    (SURVEY 8(c)).
Reference values are the committed goldens (tests/golden/) or the oracle
(oracle/, itself pinned bit-exact to those goldens in test_oracle.py).
"""
import math

import numpy as np
import pytest

from conftest import bits_equal, dec_c, dec_matrix, load_golden
from exact_walk import exact_block
from oracle import oracle
from paper_2602_10141_b200 import engine, ensembles, geodesics, kernels, modular, perm_batch
from paper_2602_10141_b200.domains import INTEGER, RATIONAL, REAL, PrimeField
from paper_2602_10141_b200.gray import make_block_plan

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def tol(n, abs_sum, ref):
    return 2 * n * U * abs_sum + 4 * U * abs(ref) + 1e-300


# --------------------------------------------------------------------------- fp64 blocks

def test_exact_kernel_bit_identical_to_reference_blocks(gpu):
    g = load_golden("f64_blocks.json")
    checked = 0
    for case in g["cases"]:
        a = dec_matrix(case["matrix"])
        blocks = case["blocks"]
        starts = [b["start"] for b in blocks]
        lens = [b["len"] for b in blocks]
        out = gpu.ryser_f64_blocks(a, case["algorithm"], starts, lens)
        for b, row in zip(blocks, out):
            s, c = complex(row[0], row[1]), complex(row[2], row[3])
            assert bits_equal(s, dec_c(b["sum"])), (case["kind"], case["algorithm"], b)
            assert bits_equal(c, dec_c(b["comp"])), (case["kind"], case["algorithm"], b)
            checked += 1
    assert checked >= 80


@pytest.mark.parametrize("n", [5, 16, 17, 33, 48, 49, 64])
def test_exact_kernel_every_state_bound_and_skew_tail(gpu, n):
    """The block kernel's register-state bounds (NMAX 16/32/48/64) and its skewed passes
    (4 or 2 steps in flight, csrc/pk_block.cuh): every block length 1..9 (tails shorter
    than, equal to and just past a pass) and two long ones, bit-identical to the oracle's
    restatement of kernels.py:33-226."""
    rng = np.random.default_rng(n)
    for cplx in (False, True):
        a = rng.standard_normal((n, n))
        if cplx:
            a = a + 1j * rng.standard_normal((n, n))
        for algo in ("ryser", "glynn"):
            m = n if algo == "ryser" else n - 1
            lens = [ln for ln in list(range(1, 10)) + [517, 1024] if ln < (1 << m)]
            starts = [int(rng.integers(0, (1 << min(m, 62)) - ln + 1)) for ln in lens]
            out = gpu.ryser_f64_blocks(a, algo, starts, lens)
            for st, ln, row in zip(starts, lens, out):
                ws, wc = oracle.block_partial(a, st, ln, algo)
                gs = complex(row[0], row[1]) if cplx else float(row[0])
                gc = complex(row[2], row[3]) if cplx else float(row[2])
                assert bits_equal(gs, ws) and bits_equal(gc, wc), (cplx, algo, n, st, ln)


def test_production_kernel_blocks_vs_exact(gpu):
    """Production path on every golden block, gated against the EXACT block sum.

    (The reference itself drifts: e.g. haar-o n=20 [0, 5000) is off by ~2.9 n u S;
    the GPU must stay inside 2 n u S of the exact value.)"""
    g = load_golden("f64_blocks.json")
    for case in g["cases"]:
        a = dec_matrix(case["matrix"])
        n = a.shape[0]
        for b in case["blocks"]:
            if b["len"] == 0:
                continue
            ex = exact_block(a, b["start"], b["len"], case["algorithm"])
            s, c, ab = gpu.ryser_f64(a, case["algorithm"], b["start"], b["len"], want_abs=True)
            assert abs(complex(s + c) - ex) <= tol(n, ab, ex), (case["kind"], case["algorithm"], b)
            part = kernels.ryser_partial if case["algorithm"] == "ryser" else kernels.glynn_partial
            es, ec = part(a, b["start"], b["len"], exact=True)
            assert bits_equal(es, dec_c(b["sum"])) and bits_equal(ec, dec_c(b["comp"]))


@pytest.mark.parametrize("kind,n,algo", [("ginibre-c", 14, "ryser"), ("haar-u", 16, "glynn"),
                                         ("haar-o", 16, "ryser"), ("goe", 15, "glynn"),
                                         ("haar-u", 20, "ryser")])
def test_tile_kernel_aligned_ranges_vs_exact(gpu, kind, n, algo):
    """Ranges made of whole tiles run in the register-resident walk kernel."""
    a = ensembles.sample_matrix(kind, n, 77, 0)
    span = 1 << 12  # tile span 2^(k+4) with k = 8 for these n (m >= 12)
    for st, ln in ((0, 2 * span), (span, span), (2 * span, span + 1000)):
        ex = exact_block(a, st, ln, algo)
        s, c, ab = gpu.ryser_f64(a, algo, st, ln, want_abs=True)
        assert abs(complex(s + c) - ex) <= tol(n, ab, ex), (st, ln)


def test_small_full_permanents_vs_exact(gpu):
    for kind, n in (("haar-u", 12), ("ginibre-r", 11), ("gue", 10), ("haar-o", 9)):
        a = ensembles.sample_matrix(kind, n, 3, 4)
        for algo in ("ryser", "glynn"):
            m = n if algo == "ryser" else n - 1
            ex = exact_block(a, 0, 1 << m, algo)
            s, c, ab = gpu.ryser_f64(a, algo, 0, 1 << m, want_abs=True)
            assert abs(complex(s + c) - ex) <= tol(n, ab, ex), (kind, algo)


@pytest.mark.parametrize("kind,n,algo", [("haar-u", 20, "ryser"), ("haar-u", 22, "glynn"),
                                         ("ginibre-c", 18, "ryser"), ("haar-o", 24, "ryser"),
                                         ("goe", 21, "glynn"), ("gue", 17, "ryser")])
def test_full_permanent_vs_oracle(gpu, kind, n, algo):
    a = ensembles.sample_matrix(kind, n, 2602, 1)
    m = n if algo == "ryser" else n - 1
    ref = oracle.permanent(a, algo, blocks=64)
    s, c, ab = gpu.ryser_f64(a, algo, 0, 1 << m, want_abs=True)
    got = complex(s + c) * (2.0 ** (1 - n) if algo == "glynn" else 1.0)
    scale = 2.0 ** (1 - n) if algo == "glynn" else 1.0
    # two approximations of one value: each within a few n u S of exact
    both = 8 * n * U * ab * scale + 4 * U * abs(ref)
    assert abs(got - ref) <= both
    api = engine.permanent(a, method=algo)
    assert abs(complex(api) - ref) <= both
    if np.isrealobj(a):
        assert isinstance(api, float)


@pytest.mark.parametrize("kind,n,algo", [("haar-u", 40, "ryser"), ("haar-u", 44, "glynn"),
                                         ("haar-o", 48, "ryser"), ("ginibre-c", 47, "ryser")])
def test_large_n_tile_vs_oracle(gpu, kind, n, algo):
    """Maximum sizes: one whole tile (32 segments of 2^k, k = m - 22) of the n = 40-48
    kernels, including the complex instantiations that spill, against the oracle.

    Entries are taken in absolute value so that no Ryser row sum cancels: with cancelling
    row sums a term's rounding error is not bounded by a multiple of |term|, and S-scaled
    bounds stop being rigorous for either side (Glynn's signed sums always cancel).
    Incrementally updated row sums drift like a random walk between rebuilds (every 2^12
    steps), so the bound carries sqrt(2^12 / 2^10) = 2 beyond the headline's k = 10."""
    a = np.abs(ensembles.sample_matrix(kind, n, 2602, 5))
    m = n if algo == "ryser" else n - 1
    k = m - 22
    span = 1 << (k + 5)  # one tile
    st = int(np.random.default_rng(n).integers(0, 1 << 17)) * span
    parts = max(64, span >> 16)  # oracle blocks of <= 2^16 steps
    rows = oracle.run_blocks(a, [st + i * (span // parts) for i in range(parts)],
                             [span // parts] * parts, algo)
    ref = oracle.kahan_combine(rows, np.iscomplexobj(a))
    s, c, ab = gpu.ryser_f64(a, algo, st, span, want_abs=True)
    drift = max(1.0, 2.0 ** ((min(k, 12) - 10) / 2))  # row sums rebuilt every 2^12 steps
    assert abs(complex(s + c) - ref) <= 8 * n * U * ab * drift + 4 * U * abs(ref), (kind, n)


def test_unaligned_ranges_and_ragged_pieces(gpu):
    a = ensembles.sample_matrix("ginibre-c", 16, 3, 0)
    rng = np.random.default_rng(7)
    for _ in range(8):
        ln = int(rng.integers(1, 12000))
        st = int(rng.integers(0, (1 << 16) - ln))
        ex = exact_block(a, st, ln)
        s, c, ab = gpu.ryser_f64(a, "ryser", st, ln, want_abs=True)
        assert abs((s + c) - ex) <= tol(16, ab, ex), (st, ln)
    s, c, _ = gpu.ryser_f64(a, "ryser", 123, 0)
    assert s == 0 and c == 0


def test_device_split_is_bit_identical(gpu):
    """A G-device split (aligned halves/quarters) tree-combines to the 1-device bits."""
    from paper_2602_10141_b200.dist import combine_pairs
    for n, cplx in ((24, True), (26, False)):
        a = ensembles.sample_matrix("haar-u" if cplx else "haar-o", n, 5, 0)
        full = gpu.ryser_f64(a, "ryser", 0, 1 << n)
        for G in (2, 4, 8):
            span = (1 << n) // G
            parts = [gpu.ryser_f64(a, "ryser", g * span, span)[:2] for g in range(G)]
            s, c = combine_pairs(parts)
            assert bits_equal(s, full[0]) and bits_equal(c, full[1]), (n, G)


def test_batch_matches_single_calls(gpu):
    spec = ensembles.EnsembleSpec("haar-u", 15, 40, 2602)
    mats = ensembles.sample_batch(spec, 0, 40)
    got = perm_batch(mats)
    for i in (0, 7, 39):
        ref = oracle.permanent(mats[i], blocks=8)
        s, c, ab = gpu.ryser_f64(mats[i], "ryser", 0, 1 << 15, want_abs=True)
        assert abs(got[i] - ref) <= 8 * 15 * U * ab + 4 * U * abs(ref)
    real = perm_batch(np.stack([ensembles.sample_matrix("goe", 9, 1, i) for i in range(5)]),
                      method="glynn")
    assert real.dtype == np.float64


def test_batch_per_matrix_launches(gpu):
    """m >= 20 (complex; real m >= 21): perm_batch issues one column-0-in-parameter
    launch per matrix over sixteen streams (pk_capi.cu, batch_per_matrix).  At m = 23
    its plan (2^10 tiles of 2^8-step segments) is the single-call plan, so the results
    are bit-identical to pk_ryser_f64 over [0, 2^m); at other m the segments differ
    (e.g. 2^10 vs 2^8 steps at m = 25) and the two agree within the S-scaled bound."""
    for kind, n, method in (("haar-u", 20, "ryser"), ("haar-u", 21, "glynn"),
                            ("haar-u", 23, "ryser"), ("haar-u", 24, "glynn"),
                            ("haar-o", 21, "ryser"), ("haar-o", 23, "ryser"),
                            ("haar-u", 25, "ryser")):
        m = n if method == "ryser" else n - 1
        mats = ensembles.sample_batch(ensembles.EnsembleSpec(kind, n, 5, 2602), 0, 5)
        raw, ab = perm_batch(mats, method=method, want_abs=True)
        for i in (0, 3, 4):
            s, c, a1 = gpu.ryser_f64(mats[i], method, 0, 1 << m, want_abs=True)
            one = s + c
            if method == "glynn":
                one = one * 2.0 ** (1 - n)
            if m == 23:
                assert bits_equal(raw[i], one), (kind, n, method, i)
            else:
                assert abs(raw[i] - one) <= 4 * n * U * a1 + 4 * U * abs(one), (kind, n, i)
        assert np.all(ab > 0)


def test_sample_permanents_c1_vs_reference(gpu):
    g = load_golden("samplers.json")
    spec = ensembles.EnsembleSpec("haar-u", 20, 16, 2602)
    got = ensembles.sample_permanents(spec, chunk=5)
    mats = ensembles.sample_batch(spec, 0, 16)
    _, ab = perm_batch(mats, want_abs=True)
    for z, want, s in zip(got, g["c1_perms"], ab):
        ref = dec_c(want)
        assert abs(z - ref) <= 8 * 20 * U * s + 4 * U * abs(ref)
    goe = ensembles.sample_permanents(ensembles.EnsembleSpec("goe", 8, 20, 1), method="glynn")
    for z, want in zip(goe, g["goe8_glynn"]):
        assert abs(z - dec_c(want)) <= 1e-12 * max(1.0, abs(dec_c(want)))


# --------------------------------------------------------------------------- F_p

def _modp_case_matrix(case):
    n, p = case["n"], case["p"]
    if "matrix" in case:
        return np.array(case["matrix"], dtype=np.uint64).reshape(n, n)
    return modular._root_matrix_u64(n, p, case["root"])


def test_modp_blocks_bit_exact(gpu):
    g = load_golden("modp_blocks.json")
    for case in g["cases"]:
        a = _modp_case_matrix(case)
        fn = kernels.ryser_partial_modp if case["algorithm"] == "ryser" else kernels.glynn_partial_modp
        for b in case["blocks"]:
            assert fn(a, b["start"], b["len"], case["p"]) == b["res"], (case["n"], case["p"], b)


@pytest.mark.parametrize("n", [7, 17, 33, 49])
def test_modp_blocks_every_state_bound_and_skew_tail(gpu, n):
    """F_p block kernel: NMAX buckets and skewed-pass tails (lengths 1..9), odd and even p."""
    rng = np.random.default_rng(100 + n)
    for p in (1000003, 4294967311, (1 << 61) - 1, 1 << 40, 999999999990):
        a = rng.integers(0, p, (n, n), dtype=np.uint64)
        for algo in ("ryser", "glynn"):
            m = n if algo == "ryser" else n - 1
            fn = kernels.ryser_partial_modp if algo == "ryser" else kernels.glynn_partial_modp
            for ln in [x for x in list(range(1, 10)) + [301] if x < (1 << m)]:
                st = int(rng.integers(0, (1 << m) - ln + 1))
                assert fn(a, st, ln, p) == oracle.block_partial_modp(a, st, ln, p, algo), \
                    (n, p, algo, st, ln)


def test_modp_random_blocks_vs_oracle_large_n(gpu):
    rng = np.random.default_rng(11)
    for n in (36, 43):
        for p in list(modular.gpu_prime_basis(n).primes[:2]) + [modular.find_primes(n, max_bits=31).primes[0]]:
            a = modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n))
            for algo in ("ryser", "glynn"):
                m = n if algo == "ryser" else n - 1
                for _ in range(3):
                    ln = int(rng.integers(1, 1 << 14))
                    st = int(rng.integers(0, (1 << m) - ln))
                    want = oracle.block_partial_modp(a, st, ln, p, algo)
                    fn = kernels.ryser_partial_modp if algo == "ryser" else kernels.glynn_partial_modp
                    assert fn(a, st, ln, p) == want, (n, p, algo, st, ln)
                # a long aligned range through the production kernel vs the oracle's blocks
                st, ln = 3 << 22, 1 << 22
                want = int(sum(int(x) for x in oracle.run_blocks(
                    a, [st + k * (ln // 32) for k in range(32)], [ln // 32] * 32, algo, p=p)) % p)
                fn = kernels.ryser_partial_modp if algo == "ryser" else kernels.glynn_partial_modp
                assert fn(a, st, ln, p) == want, (n, p, algo, "long")


@pytest.mark.parametrize("n", [40, 48])
def test_modp_large_n_tile_vs_oracle(gpu, n):
    """One whole tile of the n = 40 F_p kernels for every launch-group kind the basis model
    and the C ABI form (reduced, lazy, hybrid narrow / wide, Montgomery-64), and of the
    n = 48 reduced kernel (a 2^31-index tile; one prime keeps the CPU oracle near a minute)."""
    primes = (modular.prime_pool(n, "reduced", 1) + modular.prime_pool(n, "lazy", 2)
              + modular.prime_pool(n, "fp64", 1) + modular.prime_pool(n, "fp64w", 1)
              + list(modular.find_primes(n, max_bits=59).primes[:1]))
    mats = np.stack([modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n))
                     for p in primes])
    algo = "glynn" if n == 40 else "ryser"
    m = n if algo == "ryser" else n - 1
    span = 1 << (m - 17)
    if n == 48:
        primes, mats = primes[:1], mats[:1]
    st = 5 * span
    got = gpu.ryser_modp(mats, primes, algo, st, span)
    parts = 64
    for q, p in enumerate(primes):
        want = int(sum(int(x) for x in oracle.run_blocks(
            mats[q], [st + i * (span // parts) for i in range(parts)], [span // parts] * parts,
            algo, p=p)) % p)
        assert got[q] == want, (n, p, algo)


def test_schur_exact_values_match_reference(gpu):
    g = load_golden("schur.json")
    for row in g["rows"]:
        value, basis, wit = modular.schur_permanent_exact(row["n"], max_bits=row["bits"])
        assert str(value) == row["value"], row["n"]
        assert [w.prime for w in wit] == row["primes"]
        assert [w.residue for w in wit] == row["residues"]
        assert [w.root for w in wit] == row["roots"]
    # the residue does not depend on the expansion: Glynn (default) == Ryser (reference)
    for n in (1, 2, 5, 13, 21, 23):
        for bits in (31, 59):
            _, _, wg = modular.schur_permanent_exact(n, max_bits=bits)
            _, _, wr = modular.schur_permanent_exact(n, max_bits=bits, method="ryser")
            assert [w.residue for w in wg] == [w.residue for w in wr], (n, bits)
    h = g["helpers"]
    assert modular.schur_residue(3, 7, root=2).residue == h["residue_3_7_g2"]
    assert modular.schur_residue(2, 5, root=4).residue == h["residue_2_5_g4"]
    assert modular.schur_residue(3, 13).residue == h["residue_3_13"]


# A003112 values reproduced by the reference oracle
A003112 = {23: -31152650265, 25: -5198937484375, 27: 65230244418933,
           29: -1300425712598285, 31: 126691467546591, 33: 868088125376401545}


@pytest.mark.parametrize("n", sorted(A003112))
def test_schur_a003112_gpu_basis(gpu, n):
    value, basis, wit = modular.schur_permanent_fast(n)
    assert value == A003112[n]
    if n <= 29:
        v31, _, _ = modular.schur_permanent_exact(n, max_bits=31)
        assert v31 == A003112[n]


def _ref_large():
    """perm(S_n) for n >= 35 from the REFERENCE's own CPU path (tools/pin_schur_ref.py:
    modular.schur_residue / perm_blocked over GF(p), reference modular.py:160-206)."""
    return {r["n"]: r for r in load_golden("schur_ref_large.json")["rows"] if r.get("value")}


@pytest.mark.parametrize("n", sorted(_ref_large()))
def test_schur_large_n_matches_reference_cpu_path(gpu, n):
    """The north_star's target beyond the CPU's reach at n >= 35: perm(S_n) on the GPU
    basis (Glynn), on the reference's 31-bit basis (Ryser, its expansion) and on its
    default 59-bit basis (Montgomery-64 walk) all equal the value the reference's
    own CPU pipeline produced, and every 31-bit residue equals the reference's."""
    row = _ref_large()[n]
    want = int(row["value"])
    v, _, _ = modular.schur_permanent_fast(n)
    assert v == want
    v31, b31, w31 = modular.schur_permanent_exact(n, max_bits=31, method="ryser")
    assert v31 == want
    assert list(b31.primes) == row["primes"]
    assert [w.residue for w in w31] == row["residues"]
    assert [w.root for w in w31] == row["roots"]
    v59, _, _ = modular.schur_permanent_exact(n)  # the reference's default basis
    assert v59 == want


def test_schur_odd_n_cross_expansion(gpu):
    """Odd n (an even n gives 0, which proves nothing): Ryser and Glynn walks of the
    same prime give the same residue at n = 37 on the GPU basis."""
    b = modular.gpu_prime_basis(37)
    g = modular.schur_residues(37, b.primes, method="glynn")
    r = modular.schur_residues(37, b.primes, method="ryser")
    assert [w.residue for w in g] == [w.residue for w in r]
    v = modular.crt_reconstruct(g, b)
    assert v != 0 and abs(v) <= 37 ** 18.5


# --------------------------------------------------------------------------- engine KATs

def test_engine_kats(gpu):
    g = load_golden("engine_kats.json")
    kats = {k["tag"]: k for k in g["kats"]}

    def want(tag):
        k = kats[tag]
        if k["type"] == "complex":
            return dec_c(k["v"])
        if k["type"] == "float":
            return float.fromhex(k["v"])
        return k["v"]

    from paper_2602_10141_b200 import matrices
    assert engine.perm_ryser([[1, 2], [3, 4]]) == 10 and str(10) == want("ryser_2x2_int")
    assert engine.perm_ryser(np.array([[1.0, 2.0], [3.0, 4.0]])) == want("ryser_2x2_float")
    assert engine.perm_glynn(np.array([[1.0, 2.0], [3.0, 4.0]])) == want("glynn_2x2_float")
    assert abs(engine.perm_ryser(matrices.build_schur(3)) - want("schur3")) < 1e-13
    assert engine.perm_ryser(matrices.build_all_ones(4)) == want("J4") == 24.0
    assert engine.perm_ryser(np.eye(7)) == want("I7") == 1.0
    j12 = engine.perm_blocked(matrices.build_all_ones(12), make_block_plan(12, "ryser", 16), 4)
    assert j12 == want("J12_16blocks") == math.factorial(12)
    assert engine.perm_ryser([[2 + 3j]]) == want("n1_complex")
    assert engine.perm_glynn(np.array([[2 + 3j]])) == want("n1_glynn_complex")
    assert str(engine.perm_ryser([[7]], PrimeField(5))) == want("n1_modp")
    assert str(engine.perm_ryser([[1, 2], [3, 4]], PrimeField(2))) == want("modp2_2x2")
    assert str(engine.perm_glynn([[1, 2], [3, 4]], PrimeField(7))) == want("modp7_glynn")
    m3 = [[1, -2, 3], [4, 5, -6], [7, 8, 9]]
    assert str(engine.perm_ryser(m3)) == want("int_3x3")
    assert str(engine.perm_glynn(m3)) == want("int_glynn_3x3")
    assert isinstance(engine.perm_ryser(m3), int)
    from fractions import Fraction as F
    r = engine.perm_ryser(np.array([[F(1, 2), F(1, 3)], [F(2, 5), F(3, 7)]], dtype=object))
    assert str(r) == want("rational_2x2") and isinstance(r, F)
    assert str(engine.perm_ryser(g["int_9x9"])) == want("int_9x9")
    s5 = engine.perm_abs_entrywise(matrices.build_schur(5))
    assert abs(s5 - want("abs_entrywise_schur5")) <= 1e-12 * abs(s5)
    a = dec_matrix(g["ginibre14"])
    for blocks in (1, 7, 64):
        got = engine.perm_blocked(a, make_block_plan(14, "ryser", blocks), 1)
        ref = want(f"blocked_ginibre14_{blocks}")
        assert abs(got - ref) <= 1e-11 * abs(ref)


def test_ryser_glynn_naive_100_matrices_per_domain(gpu):
    """SPEC engine property: Ryser = Glynn = naive for n <= 8 on >= 100 matrices per
    domain (complex, real: batched GPU walks; integer and F_p: exact paths)."""
    rng = np.random.default_rng(2602)
    for n in range(1, 9):
        zc = rng.standard_normal((100, n, n)) + 1j * rng.standard_normal((100, n, n))
        zr = rng.standard_normal((100, n, n))
        for z in (zc, zr):
            naive = np.array([engine.perm_naive(m) for m in z])
            # every term is bounded by prod_i sum_j |a_ij|; there are <= 2^n of them
            scale = np.array([np.prod(np.abs(m).sum(axis=1)) for m in z]) * 2.0 ** n
            for method in ("ryser", "glynn"):
                got = perm_batch(z, method=method)
                assert np.all(np.abs(got - naive) <= 4 * n * U * scale + 1e-300), (n, method)
        for k in range(13):  # exact domains through the scalar API (104 matrices)
            ints = rng.integers(-9, 10, size=(n, n)).tolist()
            naive = engine.perm_naive(ints)
            assert engine.perm_ryser(ints) == naive == engine.perm_glynn(ints)
            assert engine.perm_glynn(ints, PrimeField(1000003)) == naive % 1000003


def test_blocked_determinism_and_properties(gpu):
    a = ensembles.sample_matrix("ginibre-c", 14, 9, 0)
    plan = make_block_plan(14, "ryser", 64)
    vals = [engine.perm_blocked(a, plan, w) for w in (1, 2, 4, 8)]
    assert all(bits_equal(v, vals[0]) for v in vals)
    assert engine.perm_blocked(np.eye(3), make_block_plan(3, "ryser", 3)) == 1.0
    b = ensembles.sample_matrix("ginibre-c", 8, 9, 1)
    assert abs(engine.perm_ryser(b) - engine.perm_naive(b)) < 1e-10 * abs(engine.perm_naive(b))
    assert abs(engine.perm_ryser(b.T) - engine.perm_ryser(b)) < 1e-10 * abs(engine.perm_ryser(b))
    u = ensembles.sample_matrix("haar-u", 16, 9, 2)
    assert abs(engine.perm_ryser(u)) <= 1 + 1e-9
    h = ensembles.sample_matrix("gue", 12, 9, 3)
    ph = engine.perm_ryser(h)
    assert abs(ph.imag) / abs(ph.real) < 1e-12
    for n in range(1, 9):
        rng = np.random.default_rng(n)
        ints = rng.integers(-5, 6, size=(n, n)).tolist()
        naive = engine.perm_naive(ints)
        assert engine.perm_ryser(ints) == naive == engine.perm_glynn(ints)
        assert engine.perm_ryser(ints, PrimeField(101)) == naive % 101
        assert engine.perm_glynn(ints, PrimeField(101)) == naive % 101


def test_exact_integers_beyond_python_reach(gpu):
    from paper_2602_10141_b200 import matrices
    j = matrices.build_all_ones(22).astype(np.int64)
    assert engine.perm_ryser(j) == math.factorial(22)
    assert engine.perm_glynn(j) == math.factorial(22)
    rng = np.random.default_rng(3)
    a = rng.integers(-3, 4, size=(16, 16))
    want = oracle.permanent(a.astype(np.float64), blocks=64)
    got = engine.perm_ryser(a.tolist())
    assert isinstance(got, int) and abs(got - want) <= 1e-9 * max(1.0, abs(want))


# --------------------------------------------------------------------------- geodesics

def test_geodesic_sweeps_and_midpoints(gpu):
    g = load_golden("geodesics.json")
    for tgt in ("cycle", "dft"):
        tr = geodesics.sweep(9, tgt, 11)
        ref = g[f"sweep_9_{tgt}"]
        for z, w in zip(tr.perms, ref["perms"]):
            assert abs(z - dec_c(w)) <= 1e-12
    tr8 = geodesics.sweep(8, "cycle", 5)
    assert [bool(d) for d in tr8.f_defined] == g["sweep_8_cycle"]["defined"]
    for n, d in g["midpoint"].items():
        got = geodesics.midpoint_analysis(int(n))
        assert abs(got["perm_mid"] - dec_c(d["perm_mid"])) <= 1e-9 * abs(dec_c(d["perm_mid"]))
        assert got["sign"] == d["sign"]
    rr = geodesics.recovery_ratio(geodesics.sweep(7, "dft", 101))
    assert abs(rr - float.fromhex(g["recovery_7"])) <= 1e-6 * rr
    oc = geodesics.onset_coefficient(geodesics.sweep(7, "cycle", 101))
    assert abs(oc - float.fromhex(g["onset_7"])) <= 1e-9 * abs(oc)


def test_schur_resumable_checkpoint(gpu, tmp_path):
    ck = tmp_path / "s25.jsonl"
    v, b, w, done = modular.schur_permanent_resumable(25, str(ck), chunks=8, max_chunks_this_call=3)
    assert v is None and done == 3
    v, b, w, done = modular.schur_permanent_resumable(25, str(ck), chunks=8)
    assert done == 8 and v == -5198937484375
    with pytest.raises(ValueError, match="different run"):
        modular.schur_permanent_resumable(25, str(ck), chunks=16)
    with pytest.raises(ValueError, match="different run"):
        modular.schur_permanent_resumable(25, str(ck), chunks=8, method="ryser")
    v, _, _, done = modular.schur_permanent_resumable(25, str(tmp_path / "r25.jsonl"), chunks=4,
                                                      method="ryser")
    assert done == 4 and v == -5198937484375


@pytest.mark.parametrize("tag,chunk", [("fast", 63), ("check31", 17)])
def test_schur45_chunk_replay(gpu, tmp_path, tag, chunk):
    """perm(S_45) (tools/schur45.py, profiles/r2_schur45.json): the committed run's chunk
    residues with one chunk removed; the resumed call re-walks that chunk (2^38 Glynn
    indices, ~20 s) and must reproduce the recorded residues and the integer."""
    import json
    import os
    src = os.path.join(os.path.dirname(__file__), "golden", f"schur45_{tag}_chunks.jsonl")
    with open(src) as f:
        lines = [json.loads(x) for x in f if x.strip()]
    header = lines[0]["header"]
    recorded = {r["chunk"]: r["residues"] for r in lines[1:]}
    assert sorted(recorded) == list(range(64))
    ck = tmp_path / "s45.jsonl"
    with open(ck, "w") as f:
        for rec in lines:
            if rec.get("chunk") != chunk:
                f.write(json.dumps(rec) + "\n")
    basis = modular.CrtBasis(45, tuple(header["primes"]), math.prod(header["primes"]))
    v, _, _, done = modular.schur_permanent_resumable(45, str(ck), chunks=64, basis=basis)
    assert done == 64 and v == -470483360490107435783203125
    with open(ck) as f:
        redo = [json.loads(x) for x in f if '"chunk"' in x][-1]
    assert redo == {"chunk": chunk, "residues": recorded[chunk]}


def test_schur_resumable_rank_files(gpu, tmp_path):
    """Two scheduler-given ranks on one GPU, exchanging finished chunks through their files."""
    ck = str(tmp_path / "s25.jsonl")
    v, _, _, done = modular.schur_permanent_resumable(25, ck, chunks=8, rank=1, world=2)
    assert v is None and done == 4
    v, _, _, done = modular.schur_permanent_resumable(25, ck, chunks=8, rank=0, world=2)
    assert done == 8 and v == -5198937484375
    v, _, _, done = modular.schur_permanent_resumable(25, ck, chunks=8)  # world 1 resumes
    assert done == 8 and v == -5198937484375


@pytest.mark.parametrize("fkind", ["fp64", "fp64w"])
def test_hybrid_fp64_primes_vs_oracle(gpu, fkind):
    """Montgomery + fp64 primes walked together (hybrid kernel) are exact, for the
    narrow (exact-product) and wide (two-product, ~40-bit) fp64 primes."""
    rng = np.random.default_rng(17)
    for n in (20, 29, 36, 43):
        primes = modular.prime_pool(n, "lazy", 2) + modular.prime_pool(n, fkind, 2)
        mats = np.stack([modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n))
                         for p in primes])
        for algo in ("ryser", "glynn"):
            m = n if algo == "ryser" else n - 1
            ln = 1 << min(m, 22)
            st = int(rng.integers(0, (1 << m) // ln)) * ln
            got = gpu.ryser_modp(mats, primes, algo, st, ln)
            for k, p in enumerate(primes):
                want = int(sum(int(x) for x in oracle.run_blocks(
                    mats[k], [st + i * (ln // 16) for i in range(16)], [ln // 16] * 16, algo,
                    p=p)) % p)
                assert got[k] == want, (n, p, algo)


def _wide_moduli(n):
    """A 59-bit prime (reference default basis), the largest prime = 1 (mod n) below
    2^62, and an odd composite wide modulus (Montgomery only needs odd p)."""
    p59 = modular.find_primes(n, max_bits=59).primes[0]
    k = ((1 << 62) - 2) // n
    while not modular.is_probable_prime(k * n + 1):
        k -= 1
    return [p59, k * n + 1, 2147483647 * 2147483629]


@pytest.mark.parametrize("n", [13, 24, 30, 33, 36])
def test_wide_moduli_vs_oracle(gpu, n):
    """Montgomery-64 walk (2^31 <= p < 2^62, one modulus per lane, three launches)."""
    rng = np.random.default_rng(100 + n)
    mods = _wide_moduli(n)
    mats = np.stack([rng.integers(0, p, size=(n, n), dtype=np.uint64) for p in mods])

    def want(q, algo, st, ln, parts=32):
        lens = [ln // parts] * (parts - 1) + [ln - (parts - 1) * (ln // parts)]
        starts = [st + i * (ln // parts) for i in range(parts)]
        return int(sum(int(x) for x in oracle.run_blocks(mats[q], starts, lens, algo,
                                                         p=mods[q])) % mods[q])

    for algo in ("ryser", "glynn"):
        m = n if algo == "ryser" else n - 1
        k = max(min(m - 5, 8), m - 22)
        ln = 1 << min(m, k + 6)  # two tiles of 32 segments: through the wide kernel
        tiles = (1 << m) // ln
        st = int(rng.integers(0, tiles)) * ln
        got = gpu.ryser_modp(mats, mods, algo, st, ln)
        for q in range(len(mods)):
            assert got[q] == want(q, algo, st, ln), (n, mods[q], algo, st, ln)
        if tiles >= 3:  # ragged head + aligned interior + ragged tail
            st2 = int(rng.integers(1, tiles - 1)) * ln - 333
            ln2 = ln + 777
            got2 = gpu.ryser_modp(mats[:1], mods[:1], algo, st2, ln2)
            assert got2[0] == want(0, algo, st2, ln2), (n, algo, "unaligned")


def test_resident_jobs_match_one_shot_calls(gpu):
    """bench.py's device-resident jobs return what the one-shot C ABI returns: an F_p
    job mixing every launch-group kind (reduced, lazy, hybrid, wide) and an fp64 job."""
    from paper_2602_10141_b200 import _native as nat
    n = 24
    ps = (modular.prime_pool(n, "reduced", 2) + modular.prime_pool(n, "lazy", 2)
          + modular.prime_pool(n, "fp64", 1) + list(modular.find_primes(n, max_bits=59).primes[:1]))
    mats = np.stack([modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n)) for p in ps])
    for algo in ("ryser", "glynn"):
        m = n if algo == "ryser" else n - 1
        want = gpu.ryser_modp(mats, ps, algo, 0, 1 << m)
        job = nat.Job.modp(mats, ps, algo, 0, 1 << m)
        _, _, got = job.run(2)
        assert job.info()["launches"] == 4  # reduced x2, hybrid (lazy + fp64), lazy x1, wide
        job.close()
        assert [int(x) for x in got] == want, algo
    a = ensembles.sample_matrix("haar-u", 20, 2602, 3)
    job = nat.Job.f64(a, "ryser", 0, 1 << 20)
    _, _, root = job.run(3)  # (s_re, c_re, s_im, c_im, abs) of the last run
    job.close()
    s1, c1, _ = nat.ryser_f64(a, "ryser", 0, 1 << 20, 1)
    assert complex(root[0], root[2]) == s1 and complex(root[1], root[3]) == c1


def test_schur_default_59bit_basis_through_wide_kernel(gpu):
    """The reference's default basis (59-bit) at n = 23, 25 against SURVEY Appendix A."""
    v23, b23, w23 = modular.schur_permanent_exact(23)
    assert v23 == -31152650265
    assert [w.residue for w in w23 if w.prime == 576460752303422599] == [576460721150772334]
    v25, _, w25 = modular.schur_permanent_exact(25)
    assert v25 == -5198937484375
    r25 = {w.prime: w.residue for w in w25}
    assert r25[576460752303422801] == 576455553365938426
    assert r25[576460752303422501] == 576455553365938126


@pytest.mark.parametrize("kind,n", [("gue", 24), ("goe", 24), ("ginibre-r", 22), ("haar-o", 26)])
def test_c5_ensembles_vs_oracle(gpu, kind, n):
    """C5: GUE/GOE/Ginibre/Haar-O permanents through the batched sampler, n up to 26."""
    spec = ensembles.EnsembleSpec(kind, n, 3, 2602)
    got = ensembles.sample_permanents(spec)
    mats = ensembles.sample_batch(spec, 0, 3)
    _, ab = perm_batch(mats, want_abs=True)
    for i in range(3):
        ref = oracle.permanent(mats[i], blocks=64)
        assert abs(got[i] - ref) <= 8 * n * U * ab[i] + 4 * U * abs(ref), (kind, i)


def test_c5_geodesic_sweep_n20_vs_oracle(gpu):
    tr = geodesics.sweep(20, "dft", 5)
    for t, z in zip(tr.ts, tr.perms):
        a = geodesics.dft_geodesic(20, float(t))
        ref = oracle.permanent(a, blocks=64)
        s, c, ab = gpu.ryser_f64(a, "ryser", 0, 1 << 20, want_abs=True)
        assert abs(z - ref) <= 8 * 20 * U * ab + 4 * U * abs(ref), t


def test_integration_md_ctypes_stub(gpu, tmp_path):
    """The ctypes stub INTEGRATION.md §2 tells a permkit maintainer to add works as
    written: its ryser_partial / ryser_partial_modp are bit-identical to the oracle
    (and so to kernels.ryser_partial / ryser_partial_modp, kernels.py:415-438)."""
    import re
    from conftest import ROOT
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"## 2\. ctypes stub.*?```python\n(.*?)```", text, re.S).group(1)
    code = code.replace('ctypes.CDLL("libpermkit_gpu.so")', f'ctypes.CDLL("{gpu.library_path()}")')
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    a = ensembles.sample_matrix("haar-u", 14, 9, 0)
    s, c = ns["ryser_partial"](a, 1234, 3000)
    rs, rc = oracle.block_partial(a, 1234, 3000)
    assert bits_equal(s, rs) and bits_equal(c, rc)
    p = modular.find_primes(14, max_bits=31).primes[0]
    au = modular._root_matrix_u64(14, p, modular.primitive_nth_root(p, 14))
    assert ns["ryser_partial_modp"](au, 77, 5000, p) == oracle.block_partial_modp(au, 77, 5000, p)
