"""Multi-device paths of the C ABI, exercised on one GPU through logical devices.

`pk_set_logical_devices(8)` makes the library report eight devices, each with its
own context (stream, buffers, lock) and host thread, mapped onto the visible
GPU(s) (permkit_gpu.h).  The per-device range / modulus splits and the combine
of the device results (pk_capi.cu: f64_range, pk_ryser_modp, pk_ryser_f64_batch)
therefore run exactly as on an 8-GPU box.  The devices never wait on each other,
so sharing one GPU only serialises them.

Gates: fp64 results bit-identical to one device for every ndev and every range
(aligned or not); F_p residues exact (equal to one device and to the oracle);
batched results independent of ndev, batch size, chunking and sub-batching.
Reference split rules: engine.py:234-236 (per-block pool), modular.py:199-204
(per-prime pool), ensembles.py:149-157 (per-sample loop).
"""
import os

import numpy as np
import pytest

from conftest import bits_equal
from oracle import oracle
from paper_2602_10141_b200 import ensembles, modular, perm_batch

pytestmark = pytest.mark.gpu


@pytest.fixture()
def logical8(gpu):
    gpu.set_logical_devices(8)
    assert gpu.device_count() == 8
    try:
        yield gpu
    finally:
        gpu.set_logical_devices(0)


def _pair_bits(x, y):
    return bits_equal(x[0], y[0]) and bits_equal(x[1], y[1])


@pytest.mark.parametrize("kind,n,algo", [("haar-u", 22, "ryser"), ("haar-o", 23, "glynn"),
                                         ("ginibre-c", 17, "ryser")])
def test_f64_device_split_bit_identical(logical8, kind, n, algo):
    gpu = logical8
    a = ensembles.sample_matrix(kind, n, 11, 0)
    m = n if algo == "ryser" else n - 1
    rng = np.random.default_rng(n)
    ranges = [(0, 1 << m), (0, 1 << (m - 1)), (1 << (m - 2), 3 << (m - 3))]
    for _ in range(3):  # unaligned: ragged head and tail pieces, cuts inside groups
        ln = int(rng.integers(1 << (m - 3), 1 << (m - 1)))
        ranges.append((int(rng.integers(1, (1 << m) - ln)), ln))
    for st, ln in ranges:
        one = gpu.ryser_f64(a, algo, st, ln, devices=1, want_abs=True)
        for nd in (2, 3, 4, 5, 8):
            got = gpu.ryser_f64(a, algo, st, ln, devices=nd, want_abs=True)
            assert _pair_bits(got, one), (kind, n, algo, st, ln, nd)
            assert got[2] == one[2]


def test_f64_split_matches_oracle_tolerance(logical8):
    """The 8-device result of a full permanent against the oracle (8 n u S)."""
    gpu = logical8
    a = ensembles.sample_matrix("haar-u", 20, 2602, 3)
    s, c, ab = gpu.ryser_f64(a, "ryser", 0, 1 << 20, devices=8, want_abs=True)
    ref = oracle.permanent(a, "ryser", blocks=64)
    assert abs((s + c) - ref) <= 8 * 20 * 2.0 ** -53 * ab + 4 * 2.0 ** -53 * abs(ref)


def _moduli(n):
    """One modulus of every launch-group / walker kind at this n."""
    red = modular.prime_pool(n, "reduced", 2)
    lazy = modular.prime_pool(n, "lazy", 2)
    fp = modular.prime_pool(n, "fp64", 1)
    fpw = modular.prime_pool(n, "fp64w", 1)
    wide = list(modular.find_primes(n, max_bits=59).primes[:1])
    return red + lazy + fp + fpw + wide + [15, 4, 2]


def _residue_mats(n, moduli, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, p, size=(n, n), dtype=np.uint64) if p > 2
                     else rng.integers(0, p, size=(n, n)).astype(np.uint64) for p in moduli])


@pytest.mark.parametrize("n,algo", [(21, "ryser"), (24, "glynn")])
def test_modp_device_split_exact(logical8, n, algo):
    gpu = logical8
    moduli = _moduli(n)
    mats = _residue_mats(n, moduli, n)
    m = n if algo == "ryser" else n - 1
    for st, ln in ((0, 1 << m), (12345, (1 << m) - 20000), (777, 1 << 14)):
        one = gpu.ryser_modp(mats, moduli, algo, st, ln, devices=1)
        for nd in (2, 3, 8):
            assert gpu.ryser_modp(mats, moduli, algo, st, ln, devices=nd) == one, (st, ln, nd)
        if ln <= 1 << 14:  # small enough for the oracle on every modulus
            for k, p in enumerate(moduli):
                assert one[k] == oracle.block_partial_modp(mats[k], st, ln, p, algo), (p, st)


def test_schur_residues_over_devices(logical8):
    """perm(S_33) (A003112) with the walk split over 8 logical devices."""
    basis = modular.gpu_prime_basis(33)
    wit = modular.schur_residues(33, basis.primes, devices=8)
    assert modular.crt_reconstruct(wit, basis) == 868088125376401545


def test_batch_independent_of_devices_and_batch_size(logical8):
    """Advisor round 1: the batched plan used to depend on the per-device batch
    size (n = 19 complex: k = 9 at 4096 matrices, 8 at 2048).  The plan now
    depends on (n, algo) only: batched == single calls, bit for bit, for every
    device count and sub-batch size."""
    gpu = logical8
    mats = ensembles.sample_batch(ensembles.EnsembleSpec("haar-u", 19, 96, 2602), 0, 96)
    ref = perm_batch(mats, devices=1)
    for nd in (2, 3, 8):
        assert np.array_equal(perm_batch(mats, devices=nd).view(np.uint64), ref.view(np.uint64))
    for lo, hi in ((0, 1), (5, 41), (41, 96)):
        assert np.array_equal(perm_batch(mats[lo:hi]).view(np.uint64), ref[lo:hi].view(np.uint64))
    for i in (0, 50, 95):
        s, c, _ = gpu.ryser_f64(mats[i], "ryser", 0, 1 << 19)
        assert bits_equal(s + c, ref[i]), i


def test_sample_permanents_chunk_invariant(logical8):
    spec = ensembles.EnsembleSpec("haar-u", 19, 300, 7)
    a = ensembles.sample_permanents(spec, chunk=300, devices=1)
    b = ensembles.sample_permanents(spec, chunk=64, devices=8)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("kind,n,method", [("haar-u", 20, "ryser"), ("haar-o", 16, "glynn")])
def test_batch_subbatches_and_stream_reuse(logical8, kind, n, method):
    """B = 40 > 16 aux streams, sub-batches of 3 (PK_BATCH_SUBBATCH): the
    per-matrix launches reuse streams and the partials / group buffers across
    sub-batches; every matrix must equal its single call."""
    gpu = logical8
    mats = ensembles.sample_batch(ensembles.EnsembleSpec(kind, n, 40, 5), 0, 40)
    ref = perm_batch(mats, method=method)
    os.environ["PK_BATCH_SUBBATCH"] = "3"
    try:
        got = perm_batch(mats, method=method)
        got8 = perm_batch(mats, method=method, devices=8)
    finally:
        del os.environ["PK_BATCH_SUBBATCH"]
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(got8.view(np.uint64), ref.view(np.uint64))
    m = n if method == "ryser" else n - 1
    for i in range(40):
        s, c, _ = gpu.ryser_f64(mats[i], method, 0, 1 << m)
        v = s + c
        if method == "glynn":
            v = v * 2.0 ** (1 - n)
        assert bits_equal(v, ref[i]), i


def test_batch_more_than_65535_matrices(gpu):
    """Advisor round 1: gridDim.y of the group fold is capped at 65535; the reduce
    now runs in slices.  70,000 real 8 x 8 matrices in one call."""
    rng = np.random.default_rng(3)
    mats = rng.standard_normal((70000, 8, 8))
    got = perm_batch(mats)
    assert np.array_equal(got[:100].view(np.uint64), perm_batch(mats[:100]).view(np.uint64))
    assert np.array_equal(got[-100:].view(np.uint64), perm_batch(mats[-100:]).view(np.uint64))
    for i in (0, 65535, 69999):
        ref = oracle.permanent(mats[i], blocks=1)
        assert abs(got[i] - ref) <= 1e-12 * max(1.0, abs(ref))


def test_tiny_batch_single_launch(gpu):
    """m < 6 (n <= 5 Ryser): every matrix is one exact piece, all in one launch."""
    rng = np.random.default_rng(4)
    mats = rng.standard_normal((500, 5, 5)) + 1j * rng.standard_normal((500, 5, 5))
    got = perm_batch(mats)
    for i in (0, 250, 499):
        s, c, _ = gpu.ryser_f64(mats[i], "ryser", 0, 32)
        assert bits_equal(s + c, got[i])


@pytest.mark.parametrize("kind,n,algo,nblocks", [("haar-u", 24, "ryser", 512),
                                                 ("haar-o", 22, "glynn", 96),
                                                 ("ginibre-c", 13, "ryser", 300)])
def test_plan_call_matches_single_range_calls(logical8, kind, n, algo, nblocks):
    """pk_ryser_f64_plan (perm_blocked's one call per plan, reference
    engine.py:213-245): every block's pair equals pk_ryser_f64 on that block, bit
    for bit, on 1 and 8 devices; uneven (make_block_plan) and irregular plans."""
    from paper_2602_10141_b200.gray import make_block_plan
    gpu = logical8
    a = ensembles.sample_matrix(kind, n, 4, 0)
    m = n if algo == "ryser" else n - 1
    plan = make_block_plan(n, algo, nblocks)
    starts = [b.start for b in plan.blocks]
    lens = [b.length for b in plan.blocks]
    rng = np.random.default_rng(n)
    cuts = np.sort(rng.choice(np.arange(1, 1 << m), size=40, replace=False))
    bounds = [0, *cuts.tolist(), 1 << m]
    irr_s, irr_l = bounds[:-1], [b - a_ for a_, b in zip(bounds[:-1], bounds[1:])]
    for st, ln in ((starts, lens), (irr_s, irr_l)):
        one, ab1 = gpu.ryser_f64_plan(a, algo, st, ln, devices=1, want_abs=True)
        eight, ab8 = gpu.ryser_f64_plan(a, algo, st, ln, devices=8, want_abs=True)
        assert np.array_equal(one.view(np.uint64), eight.view(np.uint64))
        assert np.array_equal(ab1, ab8)
        for i in list(range(0, len(st), max(1, len(st) // 17))) + [len(st) - 1]:
            s, c, ab = gpu.ryser_f64(a, algo, st[i], ln[i], want_abs=True)
            s, c = complex(s), complex(c)
            row = one[i]
            assert bits_equal(s, complex(row[0], row[1])) and bits_equal(c, complex(row[2], row[3])), i
            assert ab == ab1[i]


def test_perm_blocked_plan_vs_oracle(gpu):
    """perm_blocked through the plan call against the oracle's plan combine."""
    from paper_2602_10141_b200 import engine
    from paper_2602_10141_b200.gray import make_block_plan
    a = ensembles.sample_matrix("haar-u", 18, 9, 0)
    plan = make_block_plan(18, "ryser", 37)
    got = engine.perm_blocked(a, plan)
    ref = oracle.permanent(a, "ryser", blocks=37)
    s, c, ab = gpu.ryser_f64(a, "ryser", 0, 1 << 18, want_abs=True)
    assert abs(got - ref) <= 8 * 18 * 2.0 ** -53 * ab + 4 * 2.0 ** -53 * abs(ref)


def test_plan_call_errors_and_edges(gpu):
    """pk_ryser_f64_plan: empty plans, zero-length blocks, out-of-range blocks."""
    a = ensembles.sample_matrix("haar-u", 10, 1, 0)
    out, ab = gpu.ryser_f64_plan(a, "ryser", [], [])
    assert out.shape == (0, 4)
    out, _ = gpu.ryser_f64_plan(a, "ryser", [0, 5, 5], [5, 0, (1 << 10) - 5])
    assert np.all(out[1] == 0)
    s, c = gpu.kahan_fold(out, True)
    one = gpu.ryser_f64(a, "ryser", 0, 1 << 10)
    assert abs((s + c) - (one[0] + one[1])) < 1e-12 * abs(one[0] + one[1]) + 1e-300
    with pytest.raises(gpu.GpuError):
        gpu.ryser_f64_plan(a, "ryser", [1000], [100])  # beyond 2^10


def test_concurrent_calls_from_host_threads(gpu):
    """The reference calls its block kernels from a ThreadPoolExecutor
    (engine.py:234-236); the C ABI is reentrant (per-device lock, per-thread error
    state): eight threads mixing fp64 ranges, F_p walks and plans give exactly the
    serial results."""
    from concurrent.futures import ThreadPoolExecutor
    a = ensembles.sample_matrix("haar-u", 18, 3, 0)
    p = modular.find_primes(18, max_bits=31).primes[0]
    au = modular._root_matrix_u64(18, p, modular.primitive_nth_root(p, 18))

    def job(i):
        st, ln = 1000 * i, (1 << 15) + 37 * i
        f = gpu.ryser_f64(a, "ryser" if i % 2 else "glynn", st, ln)
        r = gpu.ryser_modp(au[None], [p], "ryser", st, ln)[0]
        pl, _ = gpu.ryser_f64_plan(a, "ryser", [st, st + ln // 2], [ln // 2, ln - ln // 2])
        return f, r, pl.tobytes()

    serial = [job(i) for i in range(24)]
    with ThreadPoolExecutor(8) as pool:
        par = list(pool.map(job, range(24)))
    for (f1, r1, p1), (f2, r2, p2) in zip(serial, par):
        assert _pair_bits(f1, f2) and r1 == r2 and p1 == p2
