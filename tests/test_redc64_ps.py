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


def _madc_hi(a, b, c, cf):
    """madc.hi.cc.u32: hi32(a b) + c + carry-in -> (32-bit result, carry-out)."""
    v = (a * b >> 32) + c + cf
    return v & M32, v >> 32


def _add(a, b, cf=0):
    """add.cc / addc.cc on 32-bit words."""
    v = a + b + cf
    return v & M32, v >> 32


def redc64_ps(x, y, p):
    """Form 2 (PK_REDC64_PS = 2): the PTX's 32-bit word steps and carry flags."""
    q0 = (-pow(p, -1, 1 << 64)) & M32
    x0, x1, y0, y1, p0, p1 = x & M32, x >> 32, y & M32, y >> 32, p & M32, p >> 32
    lo = x0 * y0
    a = x1 * y0 + x0 * y1
    assert a <= M64  # mad.wide addend
    hi = x1 * y1
    l0, l1 = lo & M32, lo >> 32
    m0 = (l0 * q0) & M32
    a = m0 * p1 + a
    assert a <= M64
    s0, s1 = a & M32, a >> 32
    _, cf = _add(l0, M32)  # carry = (l0 != 0)
    h0, cf = _madc_hi(m0, p0, l1, cf)
    s1, c = _add(s1, 0, cf)
    assert c == 0
    s0, cf = _add(s0, h0)
    s1, c = _add(s1, 0, cf)
    assert c == 0  # S < 2^64
    m1 = (s0 * q0) & M32
    r = m1 * p1 + hi
    assert r <= M64
    r0, r1 = r & M32, r >> 32
    _, cf = _add(s0, M32)  # carry = (s0 != 0)
    h1, cf = _madc_hi(m1, p0, s1, cf)
    r1, c = _add(r1, 0, cf)
    assert c == 0
    r0, cf = _add(r0, h1)
    r1, c = _add(r1, 0, cf)
    assert c == 0
    return r0 | r1 << 32


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
