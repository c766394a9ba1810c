"""The lazy Montgomery-64 walk's REDC (csrc/pk_walk64.cuh: redc64_ps), restated
step for step on 32-bit words: every 64-bit intermediate the PTX keeps in a
register pair must fit, and the output must be x y 2^-64 mod p in [0, 2p) for the
lazy walk's operand range (p < 2^60, x, y < 4p).  The GPU parity tests check the
kernel itself; this pins the bounds the word layout relies on.  Reference:
the _mulmod it replaces, kernels.py:229-247."""
import random

import pytest

M32 = (1 << 32) - 1
M64 = (1 << 64) - 1


def redc64_ps(x, y, p):
    q0 = (-pow(p, -1, 1 << 64)) & M32
    x0, x1, y0, y1, p0, p1 = x & M32, x >> 32, y & M32, y >> 32, p & M32, p >> 32
    lo = x0 * y0
    a = x1 * y0 + x0 * y1
    hi = x1 * y1
    l0, l1 = lo & M32, lo >> 32
    m0 = (l0 * q0) & M32
    a = m0 * p1 + a
    assert a <= M64  # mad.wide addend
    s = a + l1 + (m0 * p0 >> 32) + (l0 != 0)
    assert s <= M64  # carry chain ends in s1
    s0, s1 = s & M32, s >> 32
    m1 = (s0 * q0) & M32
    r = m1 * p1 + hi
    assert r <= M64
    r += s1 + (m1 * p0 >> 32) + (s0 != 0)
    assert r <= M64
    return r


@pytest.mark.parametrize("bits", [32, 40, 52, 58, 59, 60])
def test_redc64_ps_range_and_value(bits):
    rng = random.Random(bits)
    for _ in range(4000):
        p = rng.randrange(1 << (bits - 1), 1 << bits) | 1
        for x, y in ((rng.randrange(4 * p), rng.randrange(4 * p)), (4 * p - 1, 4 * p - 1),
                     (0, rng.randrange(4 * p)), (1, 1)):
            r = redc64_ps(x, y, p)
            assert r < 2 * p
            assert r % p == x * y * pow(1 << 64, -1, p) % p
