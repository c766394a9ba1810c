"""Per-block kernel seam, served by the sm_100a library.

Same names and return conventions as the reference's dispatch layer
(reference pkg/src/permkit/kernels.py:415-443), but every call runs on the GPU:

  ryser_partial / glynn_partial           fp64 block -> (sum, compensation)
  ryser_partial_modp / glynn_partial_modp F_p block  -> residue in [0, p)

``exact=True`` selects the bit-parity kernel (one GPU thread replays the
reference's numba walk operation for operation, kernels.py:33-226), so the
(sum, compensation) pair is bit-identical to the reference's.  The default is
the production kernel: the same block, evaluated by thousands of lanes in
aligned segments and tree-combined; its value agrees within the fp64 parity
tolerance but its (sum, comp) split differs.
F_p results are exact either way.
"""

from __future__ import annotations

import numpy as np

from . import _native


def backend_name() -> str:
    return "cuda-sm_100a"


def _f64_partial(a, start, length, algorithm, exact, devices):
    a = np.asarray(a)
    cplx = a.dtype == np.complex128
    if not cplx:
        a = np.ascontiguousarray(a, dtype=np.float64)
    if exact:
        row = _native.ryser_f64_blocks(a, algorithm, [start], [length])[0]
        if cplx:
            return complex(row[0], row[1]), complex(row[2], row[3])
        return float(row[0]), float(row[2])
    s, c, _ = _native.ryser_f64(a, algorithm, start, length,
                                devices or _native.default_devices())
    return s, c


def ryser_partial(a: np.ndarray, start: int, length: int, exact: bool = False,
                  devices: int | None = None):
    """Partial Ryser sum over one Gray block; returns (sum, compensation)."""
    return _f64_partial(a, start, length, "ryser", exact, devices)


def glynn_partial(a: np.ndarray, start: int, length: int, exact: bool = False,
                  devices: int | None = None):
    """Partial unscaled Glynn sum over one Gray block of sign vectors."""
    return _f64_partial(a, start, length, "glynn", exact, devices)


def _modp_partial(a, start, length, p, algorithm, devices):
    au = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return _native.ryser_modp(au[None], [int(p)], algorithm, start, length,
                              devices or _native.default_devices())[0]


def ryser_partial_modp(a: np.ndarray, start: int, length: int, p: int,
                       devices: int | None = None) -> int:
    return _modp_partial(a, start, length, p, "ryser", devices)


def glynn_partial_modp(a: np.ndarray, start: int, length: int, p: int,
                       devices: int | None = None) -> int:
    return _modp_partial(a, start, length, p, "glynn", devices)


def mulmod(a: int, b: int, p: int) -> int:
    """Modular product of the field kernels (exact big-int arithmetic on the host)."""
    return int(a) * int(b) % int(p)
