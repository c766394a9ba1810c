"""Property tests of the host-side logic (CPU only, hypothesis).

The plan, CRT and prime-selection code decide which Gray indices and which moduli
the kernels see; these properties pin their invariants independently of any golden
vector: block plans tile [0, 2^m) exactly (reference gray.py:60-79), the CRT lift
inverts residue maps inside its bound (modular.py:173-185), every prime pool
satisfies its kernel's admission rule, and the host reductions match their
definitions.
"""
import math

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2602_10141_b200 import _native, dist, gray, modular
from paper_2602_10141_b200.engine import KahanAccumulator


@settings(max_examples=60, deadline=None)
@given(n=st.integers(1, 40), algo=st.sampled_from(["ryser", "glynn"]), data=st.data())
def test_block_plan_tiles_the_range(n, algo, data):
    m = gray.iteration_exponent(n, algo)
    count = data.draw(st.integers(1, min(1 << m, 5000)))
    plan = gray.make_block_plan(n, algo, count)
    assert len(plan.blocks) == count
    pos = 0
    sizes = set()
    for b in plan.blocks:
        assert b.start == pos and b.length >= 1
        pos += b.length
        sizes.add(b.length)
    assert pos == 1 << m
    assert max(sizes) - min(sizes) <= 1


@settings(max_examples=40, deadline=None)
@given(n=st.integers(3, 40), data=st.data())
def test_crt_lift_inverts_residues(n, data):
    basis = modular.find_primes(n, max_bits=31)
    half = basis.product // 2
    x = data.draw(st.integers(-half + 1, half))
    wit = [modular.ResidueWitness(prime=p, root=0, residue=x % p) for p in basis.primes]
    assert modular.crt_reconstruct(wit, basis) == x


@settings(max_examples=30, deadline=None)
@given(n=st.integers(17, 48))
def test_prime_pools_satisfy_kernel_rules(n):
    for p in modular.prime_pool(n, "reduced", 3):
        assert p % n == 1 and p < 2 ** 31 and n * (p - 1) >= 2 ** 31
    for p in modular.prime_pool(n, "lazy", 3):
        assert p % n == 1 and n * (p - 1) < 2 ** 31 and not modular.fp64_prime_ok(p, n)
    for p in modular.prime_pool(n, "fp64", 2):
        assert p % n == 1 and modular.fp64_prime_ok(p, n)
    for p in modular.prime_pool(n, "fp64w", 2):
        assert p % n == 1 and p >= 2 ** 31 and modular.fp64w_prime_ok(p, n)
    for kind in ("reduced", "lazy", "fp64", "fp64w"):
        assert all(modular.is_probable_prime(p) for p in modular.prime_pool(n, kind, 2))


@settings(max_examples=25, deadline=None)
@given(n=st.integers(2, 48))
def test_gpu_basis_covers_the_bound(n):
    b = modular.gpu_prime_basis(n)
    assert b.product >= 4 * modular._perm_bound(n) + 1  # the reference target, modular.py:97-98
    assert all(p % n == 1 and modular.is_probable_prime(p) for p in b.primes)
    assert len(set(b.primes)) == len(b.primes)


@settings(max_examples=50, deadline=None)
@given(k=st.integers(0, 4), seed=st.integers(0, 2 ** 32 - 1))
def test_pair_tree_matches_split_combines(k, seed):
    """dist.combine_pairs on 2^k pairs equals the combine of its two halves' trees:
    the rank gather reproduces the subtree roots of a larger world."""
    rng = np.random.default_rng(seed)
    pairs = [(float(a), float(b)) for a, b in rng.standard_normal((1 << (k + 1), 2)) *
             np.exp(rng.uniform(-20, 20, ((1 << (k + 1)), 1)))]
    half = len(pairs) // 2
    left, right = dist.combine_pairs(pairs[:half]), dist.combine_pairs(pairs[half:])
    assert dist.combine_pairs(pairs) == dist.pair_combine(left, right)


@settings(max_examples=40, deadline=None)
@given(seed=st.integers(0, 2 ** 32 - 1), nb=st.integers(0, 64), cplx=st.booleans())
def test_kahan_fold_property(seed, nb, cplx):
    rng = np.random.default_rng(seed)
    rows = rng.standard_normal((nb, 4)) * np.exp(rng.uniform(-40, 40, (nb, 1)))
    if not cplx:
        rows[:, 1] = rows[:, 3] = 0.0
    acc = KahanAccumulator(complex_valued=cplx)
    for r in rows:
        acc.add(complex(r[0], r[1]) if cplx else r[0])
        acc.add(complex(r[2], r[3]) if cplx else r[2])
    s, c = _native.kahan_fold(rows, cplx)
    assert s == acc.sum and c == acc.compensation
    if nb:
        exact = math.fsum(rows[:, 0]) + math.fsum(rows[:, 2])
        assert abs((complex(s) + complex(c)).real - exact) <= 4 * 2.0 ** -53 * (
            math.fsum(np.abs(rows[:, 0])) + math.fsum(np.abs(rows[:, 2])))
