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
