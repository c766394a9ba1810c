"""TEST INFRASTRUCTURE ONLY — ctypes front end of the C restatement oracle.

``ryser_oracle.c`` restates the reference's numba block kernels
(/root/reference/pkg/src/permkit/kernels.py:33-344) in plain C compiled with
``-ffp-contract=off`` so that it is bit-identical to the reference.  It is
pinned against golden vectors generated from the reference itself
(tests/golden/, tools/make_golden.py).  Only tests/, __graft_entry__.smoke()
and bench.py (cpu_baseline and ``--impl reference``) may use this module; the
product package never imports it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "build" / "libryser_oracle.so"
_lib = None

KIND = {("ryser", True): 0, ("ryser", False): 1, ("glynn", True): 2, ("glynn", False): 3}


def build():
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        L = ctypes.CDLL(str(_SO))
        vp, u64, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        for nm in ("ork_ryser_block_cplx", "ork_ryser_block_real", "ork_glynn_block_cplx",
                   "ork_glynn_block_real"):
            f = getattr(L, nm)
            f.restype = None
            f.argtypes = [vp, i, u64, u64, vp]
        for nm in ("ork_ryser_block_modp", "ork_glynn_block_modp"):
            f = getattr(L, nm)
            f.restype = u64
            f.argtypes = [vp, i, u64, u64, u64]
        L.ork_mulmod.restype = u64
        L.ork_mulmod.argtypes = [u64, u64, u64]
        L.ork_run_blocks.restype = i
        L.ork_run_blocks.argtypes = [i, vp, i, vp, vp, i, u64, i, vp, vp]
        _lib = L
    return _lib


def _arr(a, cplx):
    return np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)


def block_partial(a, start: int, length: int, algorithm: str = "ryser"):
    """(sum, comp) of one block, like kernels.ryser_partial / glynn_partial."""
    cplx = np.iscomplexobj(a)
    a = _arr(a, cplx)
    out = np.zeros(4)
    fn = {0: lib().ork_ryser_block_cplx, 1: lib().ork_ryser_block_real,
          2: lib().ork_glynn_block_cplx, 3: lib().ork_glynn_block_real}[KIND[(algorithm, cplx)]]
    fn(a.ctypes.data, a.shape[0], int(start), int(length), out.ctypes.data)
    if cplx:
        return complex(out[0], out[1]), complex(out[2], out[3])
    return float(out[0]), float(out[2])


def block_partial_modp(a, start: int, length: int, p: int, algorithm: str = "ryser") -> int:
    """Residue of one block, like kernels.ryser_partial_modp / glynn_partial_modp."""
    au = np.ascontiguousarray(np.asarray(a, dtype=object).astype(np.uint64))
    fn = lib().ork_ryser_block_modp if algorithm == "ryser" else lib().ork_glynn_block_modp
    return int(fn(au.ctypes.data, au.shape[0], int(start), int(length), int(p)))


def mulmod(a: int, b: int, p: int) -> int:
    return int(lib().ork_mulmod(a, b, p))


def run_blocks(a, starts, lens, algorithm="ryser", p=None, threads=None):
    """Multithreaded block walk (CPU baseline); returns per-block results."""
    threads = threads or os.cpu_count() or 1
    s = np.ascontiguousarray(starts, dtype=np.uint64)
    ln = np.ascontiguousarray(lens, dtype=np.uint64)
    nb = len(s)
    if p is None:
        cplx = np.iscomplexobj(a)
        a = _arr(a, cplx)
        out = np.zeros((nb, 4))
        lib().ork_run_blocks(KIND[(algorithm, cplx)], a.ctypes.data, a.shape[0], s.ctypes.data,
                             ln.ctypes.data, nb, 0, threads, out.ctypes.data, None)
        return out
    au = np.ascontiguousarray(np.asarray(a, dtype=object).astype(np.uint64))
    out = np.zeros(nb, dtype=np.uint64)
    kind = 4 if algorithm == "ryser" else 5
    lib().ork_run_blocks(kind, au.ctypes.data, au.shape[0], s.ctypes.data, ln.ctypes.data, nb,
                         int(p), threads, None, out.ctypes.data)
    return out


def kahan_combine(partials, cplx: bool):
    """engine._run_plan's ordered combine: add(s); add(c) per block (engine.py:240-245)."""
    sr = cr = si = ci = 0.0

    def step(s, c, v):
        t = s + v
        if abs(s) >= abs(v):
            c += (s - t) + v
        else:
            c += (v - t) + s
        return t, c

    for row in partials:
        s = complex(row[0], row[1])
        c = complex(row[2], row[3])
        for z in (s, c):
            sr, cr = step(sr, cr, z.real)
            if cplx:
                si, ci = step(si, ci, z.imag)
    return complex(sr + cr, si + ci) if cplx else sr + cr


def permanent(a, algorithm="ryser", blocks=1, threads=None):
    """Full permanent via an even block plan (make_block_plan semantics, gray.py:60-79)."""
    a = np.asarray(a)
    n = a.shape[0]
    m = n if algorithm == "ryser" else n - 1
    total = 1 << m
    base, extra = divmod(total, blocks)
    lens = [base + (1 if k < extra else 0) for k in range(blocks)]
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    out = run_blocks(a, starts, lens, algorithm, threads=threads)
    v = kahan_combine(out, np.iscomplexobj(a))
    if algorithm == "glynn":
        v = v * 2.0 ** (1 - n)
    return v


def permanent_modp(a, p: int, algorithm="ryser", blocks=64, threads=None) -> int:
    a = np.asarray(a, dtype=object)
    n = a.shape[0]
    m = n if algorithm == "ryser" else n - 1
    total = 1 << m
    blocks = min(blocks, total)
    base, extra = divmod(total, blocks)
    lens = [base + (1 if k < extra else 0) for k in range(blocks)]
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    out = run_blocks(a, starts, lens, algorithm, p=p, threads=threads)
    s = sum(int(x) for x in out) % p
    if algorithm == "glynn":
        s = s * pow(pow(2, n - 1, p), -1, p) % p
    return s
