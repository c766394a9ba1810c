"""Host-side logic that needs no GPU: plans, domains, accumulators, CRT helpers,
samplers, geodesic matrices, input validation and the C-ABI library surface.

Golden values come from the reference (tests/golden/, tools/make_golden.py).
"""
import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT, bits_equal, dec_c, dec_matrix, load_golden
from paper_2602_10141_b200 import _native, engine, ensembles, geodesics, gray, matrices, modular
from paper_2602_10141_b200.domains import (COMPLEX, INTEGER, RATIONAL, REAL, PrimeField,
                                           domain_by_name, infer_domain)


# --------------------------------------------------------------------------- C ABI

def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "permkit_gpu.h").read_text()
    declared = set(re.findall(r"\b(pk_[a-z0-9_]+)\s*\(", header))
    declared -= {"pk_job"}
    lib = ctypes.CDLL(str(_native.library_path()))
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.exported_symbols()) <= declared
    assert len(declared) >= 15


def test_library_reports_no_device_without_gpu_or_a_device_count():
    n = _native.device_count()
    assert n >= 0
    assert _native.lib().pk_version() == 100
    assert _native.lib().pk_max_n() == 48


def test_no_cpu_fallback_when_no_gpu():
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_native.GpuError):
        engine.perm_ryser(np.eye(4))
    with pytest.raises(_native.GpuUnavailableError):
        _native.require_gpu()


# --------------------------------------------------------------------------- gray

def test_gray_code_and_flip_bits():
    for b in range(1, 2000):
        diff = gray.gray_code(b) ^ gray.gray_code(b - 1)
        assert diff == 1 << gray.gray_flip_bit(b)
    with pytest.raises(ValueError):
        gray.gray_flip_bit(0)


def test_block_plans_match_reference_kats():
    kats = {k["tag"]: k for k in load_golden("engine_kats.json")["kats"]}
    for blocks in (2, 3):
        plan = gray.make_block_plan(3, "ryser", blocks)
        assert str([[b.start, b.length] for b in plan.blocks]) == kats[f"plan_3_{blocks}"]["v"]
    p = gray.make_block_plan(20, "glynn", 7)
    assert p.total == 1 << 19 and all(b.length in (74898, 74899) for b in p.blocks)
    with pytest.raises(ValueError, match="too many blocks"):
        gray.make_block_plan(3, "ryser", 9)
    with pytest.raises(ValueError, match="block_count must be >= 1"):
        gray.make_block_plan(3, "ryser", 0)
    with pytest.raises(ValueError, match="unknown algorithm"):
        gray.iteration_exponent(3, "laplace")


def test_block_start_state_matches_walk():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((6, 6))
    st = gray.block_start_state(a, gray.GrayBlock(5, 1), "ryser")
    code = gray.gray_code(5)
    want = sum(a[:, j] for j in range(6) if (code >> j) & 1)
    np.testing.assert_allclose(st, want)
    st = gray.block_start_state(a, gray.GrayBlock(4, 1), "glynn")
    code = gray.gray_code(4)
    want = a[0] + sum((-a[i] if (code >> (i - 1)) & 1 else a[i]) for i in range(1, 6))
    np.testing.assert_allclose(st, want)


# --------------------------------------------------------------------------- domains

def test_domains_and_inference():
    assert infer_domain(np.zeros((2, 2), complex)) is COMPLEX
    assert infer_domain(np.zeros((2, 2))) is REAL
    assert infer_domain(np.zeros((2, 2), int)) is INTEGER
    assert infer_domain(np.array([[Fraction(1, 2)]], dtype=object)) is RATIONAL
    with pytest.raises(TypeError):
        infer_domain(np.zeros((2, 2), bool))
    assert domain_by_name("prime", 7).p == 7
    with pytest.raises(ValueError, match="needs a modulus"):
        domain_by_name("prime")
    with pytest.raises(ValueError, match=r"modulus must be a prime in \[2, 2\^62\)"):
        PrimeField(1)
    f = PrimeField(13)
    assert f.div_pow2(f.mul(5, 4), 2) == 5
    with pytest.raises(ValueError, match="GF\\(2\\)"):
        PrimeField(2).div_pow2(1, 1)


def test_kahan_accumulator_semantics():
    acc = engine.KahanAccumulator(complex_valued=True)
    for v in (1e16 + 0j, 1.0 + 1e16j, -1e16 + 0j, 1j):
        acc.add(v)
    assert acc.value == complex(1.0, 1e16 + 1.0)
    r = engine.KahanAccumulator()
    for v in (1.0, 1e100, 1.0, -1e100):
        r.add(v)
    assert r.value == 2.0


def test_input_validation_matches_reference_messages():
    with pytest.raises(ValueError, match="matrix must be square"):
        engine.perm_ryser([[1, 2, 3], [4, 5, 6]])
    with pytest.raises(ValueError, match="empty matrix"):
        engine.perm_ryser(np.zeros((0, 0)))
    with pytest.raises(engine.LimitError, match="exceeds the n <= 48 range"):
        engine.perm_ryser(np.eye(49, dtype=complex))
    # real fp64 walks go to n = 63 (Ryser) / 64 (Glynn), beyond the reference's 40
    with pytest.raises(engine.LimitError, match="exceeds the n <= 63 range of real ryser"):
        engine.perm_ryser(np.eye(64))
    with pytest.raises(engine.LimitError, match="exceeds the n <= 64 range of real glynn"):
        engine.perm_glynn(np.eye(65))
    with pytest.raises(engine.LimitError, match="exceeds the n <= 25 range"):
        engine.perm_abs_entrywise(np.eye(26))
    with pytest.raises(engine.LimitError, match="oracle dimension exceeded"):
        engine.perm_naive(np.eye(12))
    with pytest.raises(ValueError, match="division by two unavailable in GF\\(2\\)"):
        engine.perm_glynn([[1, 2], [3, 4]], PrimeField(2))
    with pytest.raises(ValueError, match="unknown method"):
        engine.permanent(np.eye(2), method="laplace")
    plan = gray.make_block_plan(4, "ryser", 2)
    with pytest.raises(ValueError, match="plan dimension does not match matrix"):
        engine.perm_blocked(np.eye(3), plan)


def test_perm_naive_reference_kats():
    kats = {k["tag"]: k for k in load_golden("engine_kats.json")["kats"]}
    g = load_golden("engine_kats.json")
    assert str(engine.perm_naive(g["int_9x9"])) == kats["int_9x9_naive"]["v"]
    assert engine.perm_naive([[1, 2], [3, 4]]) == 10
    assert engine.perm_naive([[1, 2], [3, 4]], PrimeField(7)) == 3


# --------------------------------------------------------------------------- modular

def test_modular_helpers_match_reference():
    h = load_golden("schur.json")["helpers"]
    assert list(modular.find_primes(3, ascending=True).primes) == h["find_primes_3_asc"]
    assert list(modular.find_primes(20, max_bits=31).primes) == h["find_primes_20_31"]
    assert list(modular.find_primes(36, max_bits=31).primes) == h["find_primes_36_31"]
    assert list(modular.find_primes(43, max_bits=31).primes) == h["find_primes_43_31"]
    assert list(modular.find_primes(36).primes) == h["find_primes_36_59"]
    assert modular.primitive_nth_root(7, 3) == h["root_7_3"]
    assert modular.primitive_nth_root(13, 3) == h["root_13_3"]
    assert modular.primitive_nth_root(13, 3, skip=1) == h["root_13_3_skip1"]
    for x, want in h["is_prime"].items():
        assert modular.is_probable_prime(int(x)) == want, x
    for n, b in h["perm_bound"].items():
        assert modular._perm_bound(int(n)) == b


def test_crt_round_trip_and_basis_checks():
    basis = modular.find_primes(9, max_bits=31)
    rng = np.random.default_rng(4)
    half = basis.product // 2
    for _ in range(100):
        x = int(rng.integers(-2**62, 2**62)) * int(rng.integers(1, 2**20))
        x = max(-half + 1, min(half, x))
        w = [modular.ResidueWitness(p, 0, x % p) for p in basis.primes]
        assert modular.crt_reconstruct(w, basis) == x
    w = [modular.ResidueWitness(4, 2, 0), modular.ResidueWitness(3, 1, 1)]
    with pytest.raises(ValueError, match="basis mismatch"):
        modular.crt_reconstruct(w, basis)
    with pytest.raises(ValueError, match="does not cover"):
        modular.CrtBasis(n=9, primes=(7,), product=7)
    with pytest.raises(ValueError, match="exact Schur permanents are supported"):
        modular.schur_permanent_exact(49)


def _basis_kinds(b, n):
    return [("fp64w" if p >= 2 ** 31 and modular.fp64w_prime_ok(p, n) else
             "fp64" if modular.fp64_prime_ok(p, n) else
             "lazy" if n * (p - 1) < 2 ** 31 else "red") for p in b.primes]


def test_gpu_prime_basis_properties():
    for n in (2, 13, 17, 30, 35, 36, 37, 41, 43, 48):
        b = modular.gpu_prime_basis(n)
        for p in b.primes:
            assert (p - 1) % n == 0 and modular.is_probable_prime(p)
            assert p < 2 ** 31 or modular.fp64w_prime_ok(p, n)
        assert b.product > 4 * modular._perm_bound(n) + 1
        k = _basis_kinds(b, n)
        cost = modular.basis_walk_seconds(n, k.count("red"), k.count("lazy"), k.count("fp64"),
                                          k.count("fp64w"))
        # no worse than the reference-style all-31-bit basis
        ref31 = len(modular.find_primes(n, max_bits=31).primes)
        assert cost <= modular.basis_walk_seconds(n, ref31, 0, 0) + 1e-12
        assert k.count("fp64w") <= k.count("lazy")  # every wide fp64 prime has a partner
    assert 3 <= len(modular.gpu_prime_basis(36).primes) <= 4
    assert modular._launch_groups(43, 4, 0, 0) == [("red", 3), ("red", 1)]
    assert modular._launch_groups(36, 0, 2, 2) == [("hyb", 2), ("hyb", 2)]
    assert modular._launch_groups(36, 1, 1, 0, 1) == [("hybw", 2), ("red", 1)]
    assert modular._launch_groups(36, 0, 0, 0, 1) == [("wide", 1)]
    for kind in ("reduced", "lazy", "fp64", "fp64w"):
        pool = modular.prime_pool(36, kind, 3)
        assert len(pool) == 3 and pool == sorted(pool, reverse=True)
    assert all(p >= 2 ** 31 and 36 * 36 * p <= 2 ** 50 for p in modular.prime_pool(36, "fp64w", 3))


def test_integer_crt_primes_cover_bound():
    ps = engine.integer_crt_primes(10, 10 ** 40)
    assert np.prod([float(p) for p in ps]) > 2e40
    assert all(10 * (p - 1) < 2 ** 31 and p % 2 for p in ps)


# --------------------------------------------------------------------------- samplers

def test_sampler_bit_identical_to_reference():
    g = load_golden("samplers.json")
    for m in g["matrices"]:
        a = ensembles.sample_matrix(m["kind"], m["n"], m["seed"], m["index"])
        b = dec_matrix(m["matrix"])
        assert a.tobytes() == b.astype(a.dtype).tobytes(), (m["kind"], m["index"])
    got = ensembles.RngStream(9, 4).normals(11)
    assert [float.fromhex(v) for v in g["normals"]] == list(got)
    got = ensembles.RngStream(9, 5).uniforms(5)
    assert [float.fromhex(v) for v in g["uniforms"]] == list(got)
    a0 = ensembles.sample_matrix("haar-u", 20, 2602, 0)
    assert a0.tobytes() == dec_matrix(g["c1_first_matrix"]).tobytes()


def test_sample_batch_thread_invariant():
    spec = ensembles.EnsembleSpec("haar-u", 6, 9, 17)
    a = ensembles.sample_batch(spec, 0, 9, threads=1)
    b = ensembles.sample_batch(spec, 0, 9, threads=4)
    assert a.tobytes() == b.tobytes()
    with pytest.raises(ValueError, match="unknown ensemble"):
        ensembles.EnsembleSpec("wishart", 3, 1, 0)
    with pytest.raises(ValueError, match="n and count must be >= 1"):
        ensembles.EnsembleSpec("gue", 0, 1, 0)
    with pytest.raises(ValueError, match="spec is not GUE"):
        ensembles.sample_gue(ensembles.EnsembleSpec("goe", 3, 1, 0))


def test_sampler_pool_only_for_spawn_safe_mains(tmp_path):
    """A spawn child re-runs an unguarded __main__ script, so the pool is skipped there."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    body = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2602_10141_b200 import ensembles as e\n" % root)
    unguarded = tmp_path / "u.py"
    unguarded.write_text(body + "print(e._spawn_safe())\n")
    guarded = tmp_path / "g.py"
    guarded.write_text(body + 'if __name__ == "__main__":\n    print(e._spawn_safe())\n')
    out = [subprocess.run([sys.executable, str(f)], capture_output=True, text=True,
                          timeout=120).stdout.strip() for f in (unguarded, guarded)]
    assert out == ["False", "True"]


def test_sample_batch_process_pool_bit_identical():
    """Large batches go through the spawn process pool; same bytes as one process."""
    for kind in ("haar-u", "goe"):
        spec = ensembles.EnsembleSpec(kind, 7, 700, 2602)
        a = ensembles.sample_batch(spec, 5, 705, threads=1)
        b = ensembles.sample_batch(spec, 5, 705, threads=3)
        assert a.shape == (700, 7, 7) and a.tobytes() == b.tobytes()


# --------------------------------------------------------------------------- geodesics / matrices

def test_geodesic_matrices_match_reference():
    g = load_golden("geodesics.json")
    pairs = [(geodesics.cycle_geodesic(7, 0.3), g["cycle_7_03"]),
             (geodesics.dft_geodesic(7, 0.5), g["dft_7_05"]),
             (geodesics.cycle_geodesic_real(7, 0.3), g["cycle_real_7_03"]),
             (geodesics.cycle_geodesic_real(6, 0.3), g["cycle_real_6_03"])]
    for got, want in pairs:
        np.testing.assert_allclose(got, dec_matrix(want), rtol=0, atol=1e-15)
    assert np.array_equal(geodesics.cycle_geodesic(5, 1.0), matrices.build_cycle(5))
    assert np.array_equal(geodesics.dft_geodesic(5, 0.0), np.eye(5))
    with pytest.raises(ValueError, match="t must lie"):
        geodesics.cycle_geodesic(5, 1.5)
    with pytest.raises(ValueError, match="steps must be >= 2"):
        geodesics.sweep(5, "cycle", 1)


def test_matrix_builders():
    s = matrices.build_schur(6, normalized=True)
    assert matrices.unitarity_defect(s) < 1e-14
    c = matrices.build_cycle(4)
    assert c[1, 0] == 1 and c[0, 3] == 1 and c.sum() == 4
    assert matrices.lu_log_abs_det(np.zeros((3, 3)))[0] == float("-inf")
    with pytest.raises(ValueError):
        matrices.build_schur(0)


def test_device_base_validation():
    _native.set_device_base(0)
    with pytest.raises(_native.GpuError):
        _native.set_device_base(_native.device_count() + 3)
    _native.set_device_base(0)


def test_kahan_fold_matches_kahan_accumulator():
    """pk_kahan_fold (C, in the library; no device needed) is engine._run_plan's
    ordered combine: bit-identical to KahanAccumulator add(s); add(c) per block
    (reference engine.py:33-73, 240-245)."""
    import numpy as np

    from paper_2602_10141_b200 import _native
    from paper_2602_10141_b200.engine import KahanAccumulator
    rng = np.random.default_rng(5)
    for cplx in (True, False):
        rows = rng.standard_normal((300, 4)) * np.exp(rng.uniform(-30, 30, (300, 1)))
        if not cplx:
            rows[:, 1] = rows[:, 3] = 0.0
        acc = KahanAccumulator(complex_valued=cplx)
        for r in rows:
            acc.add(complex(r[0], r[1]) if cplx else r[0])
            acc.add(complex(r[2], r[3]) if cplx else r[2])
        s, c = _native.kahan_fold(rows, cplx)
        assert s == acc.sum and c == acc.compensation


def test_kahan_fold_empty():
    import numpy as np

    from paper_2602_10141_b200 import _native
    assert _native.kahan_fold(np.zeros((0, 4)), True) == (0j, 0j)
    assert _native.kahan_fold(np.zeros((0, 4)), False) == (0.0, 0.0)
