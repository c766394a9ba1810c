"""Exact (big-integer) Gray-walk sums for tolerance checks in tests.

Every float64 entry is an integer multiple of 2^-E for a common E, so a block
sum of the Ryser / Glynn expansion is computed exactly with Python integers
(Gaussian integers for complex input; exact incremental Gray updates) and
rounded once at the end.  The GPU and the reference are both measured against
this value (SURVEY 8(c) / Appendix C method).
"""
import math
from fractions import Fraction

import numpy as np


def _scale(vals):
    e = 0
    for v in vals:
        if v != 0:
            _, ex = math.frexp(v)
            e = max(e, 53 - ex)
    return e


def exact_block(a, start, length, algorithm="ryser"):
    """Exact signed term sum over Gray indices [start, start+length) (Glynn unscaled)."""
    a = np.asarray(a)
    cplx = np.iscomplexobj(a)
    n = a.shape[0]
    re = a.real.astype(np.float64)
    im = a.imag.astype(np.float64) if cplx else np.zeros_like(re)
    E = _scale(list(re.ravel()) + list(im.ravel()))
    R = [[int(Fraction(float(re[i, j])) * (1 << E)) for j in range(n)] for i in range(n)]
    I = [[int(Fraction(float(im[i, j])) * (1 << E)) for j in range(n)] for i in range(n)]
    g = start ^ (start >> 1)
    if algorithm == "ryser":
        sr = [sum(R[i][j] for j in range(n) if (g >> j) & 1) for i in range(n)]
        si = [sum(I[i][j] for j in range(n) if (g >> j) & 1) for i in range(n)]
        neg = (n - bin(g).count("1")) & 1
    else:
        sr = [R[0][j] + sum((-R[i][j] if (g >> (i - 1)) & 1 else R[i][j]) for i in range(1, n))
              for j in range(n)]
        si = [I[0][j] + sum((-I[i][j] if (g >> (i - 1)) & 1 else I[i][j]) for i in range(1, n))
              for j in range(n)]
        neg = bin(g).count("1") & 1
    tot_r = tot_i = 0
    idx = start
    for step in range(length):
        pr, pi = 1, 0
        if cplx:
            for x, y in zip(sr, si):
                pr, pi = pr * x - pi * y, pr * y + pi * x
        else:
            for x in sr:
                pr *= x
        if neg:
            tot_r -= pr
            tot_i -= pi
        else:
            tot_r += pr
            tot_i += pi
        if step + 1 < length:
            idx += 1
            b = (idx & -idx).bit_length() - 1
            on = not ((g >> b) & 1)
            if algorithm == "ryser":
                for i in range(n):
                    if on:
                        sr[i] += R[i][b]
                        si[i] += I[i][b]
                    else:
                        sr[i] -= R[i][b]
                        si[i] -= I[i][b]
            else:
                for j in range(n):
                    if on:
                        sr[j] -= 2 * R[b + 1][j]
                        si[j] -= 2 * I[b + 1][j]
                    else:
                        sr[j] += 2 * R[b + 1][j]
                        si[j] += 2 * I[b + 1][j]
            g ^= 1 << b
            neg ^= 1
    den = 1 << (E * n)
    vr = float(Fraction(tot_r, den))
    if cplx:
        return complex(vr, float(Fraction(tot_i, den)))
    return vr
