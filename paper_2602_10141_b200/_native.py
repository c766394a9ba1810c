"""ctypes binding of the C-ABI library ``_lib/libpermkit_gpu.so``.

The library is the only execution path for permanents in this package: there
is deliberately no CPU fallback.  If the shared object is missing or no CUDA
device is visible, every call raises :class:`GpuUnavailableError` instead of
silently computing on the host.

Entry points mirror include/permkit_gpu.h one to one.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libpermkit_gpu.so"
# experiment variants (tools/build_variant.py) only; the product library is _LIB_PATH
if os.environ.get("PERMKIT_GPU_LIB"):
    _LIB_PATH = Path(os.environ["PERMKIT_GPU_LIB"]).resolve()

_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p

PK_ALGO = {"ryser": 0, "glynn": 1}


class GpuUnavailableError(RuntimeError):
    """The CUDA library or a CUDA device is not available (no CPU fallback)."""


class GpuError(RuntimeError):
    """A library call failed; carries the library's status code."""

    def __init__(self, status: int, message: str):
        super().__init__(f"permkit_gpu error {status}: {message}")
        self.status = status
        self.message = message


_lock = threading.Lock()
_lib = None


def library_path() -> Path:
    return _LIB_PATH


def _bind(lib):
    P = ctypes.POINTER
    sigs = {
        "pk_last_error": (ctypes.c_char_p, []),
        "pk_device_count": (_int, []),
        "pk_set_device_base": (_int, [_int]),
        "pk_set_logical_devices": (_int, [_int]),
        "pk_version": (_int, []),
        "pk_max_n": (_int, []),
        "pk_ryser_f64": (_int, [_vp, _int, _int, _int, _u64, _u64, _int, P(_dbl), P(_dbl)]),
        "pk_ryser_f64_blocks": (_int, [_vp, _int, _int, _int, _vp, _vp, _int, _int, _vp]),
        "pk_ryser_f64_plan": (_int, [_vp, _int, _int, _int, _vp, _vp, _int, _int, _vp, _vp]),
        "pk_ryser_f64_batch": (_int, [_vp, _int, _int, _int, _int, _int, _vp, _vp]),
        "pk_ryser_modp": (_int, [_vp, _vp, _int, _int, _int, _u64, _u64, _int, _vp]),
        "pk_job_f64_create": (_int, [_int, _vp, _int, _int, _int, _u64, _u64, P(_vp)]),
        "pk_job_modp_create": (_int, [_int, _vp, _vp, _int, _int, _int, _u64, _u64, P(_vp)]),
        "pk_job_run": (_int, [_vp, _int, ctypes.c_size_t, P(_dbl), P(_dbl), _vp, _vp]),
        "pk_job_info": (_int, [_vp, _vp]),
        "pk_job_groups": (_int, [_vp, _vp, _vp, _vp, _int]),
        "pk_job_destroy": (None, [_vp]),
        "pk_measure_peaks": (_int, [_int, _vp, _int]),
        "pk_peak_names": (ctypes.c_char_p, []),
        "pk_measure_latencies": (_int, [_int, _vp, _int]),
        "pk_latency_names": (ctypes.c_char_p, []),
        "pk_kahan_fold": (_int, [_vp, _int, _int, _vp]),
        "pk_measure_mix_ceilings": (_int, [_int, _vp, _int]),
        "pk_mix_names": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def exported_symbols():
    """Names of the C-ABI entry points this binding requires."""
    return [
        "pk_last_error", "pk_device_count", "pk_set_device_base", "pk_set_logical_devices",
        "pk_version", "pk_max_n", "pk_ryser_f64",
        "pk_ryser_f64_blocks", "pk_ryser_f64_plan", "pk_ryser_f64_batch", "pk_ryser_modp", "pk_job_f64_create",
        "pk_job_modp_create", "pk_job_run", "pk_job_info", "pk_job_groups", "pk_job_destroy",
        "pk_measure_peaks", "pk_peak_names", "pk_measure_latencies", "pk_latency_names",
        "pk_kahan_fold", "pk_measure_mix_ceilings", "pk_mix_names",
    ]


def load_library():
    """Load (once) and return the ctypes library; raises if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise GpuUnavailableError(
                    f"{_LIB_PATH} is not built; run __graft_entry__.build() "
                    "(make -C paper_2602_10141_b200/csrc)")
            _lib = _bind(ctypes.CDLL(str(_LIB_PATH)))
            base = os.environ.get("PERMKIT_GPU_DEVICE_BASE", "").strip()
            if base:
                st = _lib.pk_set_device_base(int(base))
                if st != 0:
                    raise GpuError(st, _lib.pk_last_error().decode(errors="replace"))
        return _lib


def lib():
    return load_library()


def _check(status: int):
    if status != 0:
        msg = lib().pk_last_error().decode(errors="replace")
        raise GpuError(status, msg)


def device_count() -> int:
    n = lib().pk_device_count()
    if n < 0:
        _check(n)
    return n


def set_device_base(base: int):
    """Logical device 0 of every call becomes physical device ``base`` (one process per GPU)."""
    _check(lib().pk_set_device_base(int(base)))


def set_logical_devices(count: int):
    """Test / measurement hook: report ``count`` devices, logical device d on
    visible GPU d mod (visible GPUs); 0 turns it off (permkit_gpu.h)."""
    _check(lib().pk_set_logical_devices(int(count)))


def require_gpu():
    if device_count() < 1:
        raise GpuUnavailableError("no CUDA device visible; the GPU engine has no CPU fallback")


def default_devices() -> int:
    env = os.environ.get("PERMKIT_GPU_DEVICES", "").strip()
    if env:
        return max(1, int(env))
    return 1


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def ryser_f64(a: np.ndarray, algo: str, start: int, length: int, devices: int = 1,
              want_abs: bool = False):
    """One matrix over [start, start+length); returns (sum, comp, abs_sum)."""
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    out = (_dbl * 4)()
    ab = _dbl(0.0)
    _check(lib().pk_ryser_f64(_ptr(a), a.shape[0], int(cplx), PK_ALGO[algo], int(start),
                              int(length), int(devices), out,
                              ctypes.byref(ab) if want_abs else None))
    if cplx:
        return complex(out[0], out[1]), complex(out[2], out[3]), ab.value
    return out[0], out[2], ab.value


def ryser_f64_blocks(a: np.ndarray, algo: str, starts, lens, device: int = 0) -> np.ndarray:
    """Bit-exact per-block partials; returns float64 array [nblocks, 4]."""
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    s = np.ascontiguousarray(starts, dtype=np.uint64)
    ln = np.ascontiguousarray(lens, dtype=np.uint64)
    out = np.zeros((len(s), 4), dtype=np.float64)
    _check(lib().pk_ryser_f64_blocks(_ptr(a), a.shape[0], int(cplx), PK_ALGO[algo], _ptr(s),
                                     _ptr(ln), len(s), int(device), _ptr(out)))
    return out


def ryser_f64_plan(a: np.ndarray, algo: str, starts, lens, devices: int = 1,
                   want_abs: bool = False):
    """Per-block (sum, comp) pairs of one matrix over a block plan in one call;
    returns ([nblocks, 4] float64 {s_re, s_im, c_re, c_im}, [nblocks] abs or None)."""
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    s = np.ascontiguousarray(starts, dtype=np.uint64)
    ln = np.ascontiguousarray(lens, dtype=np.uint64)
    out = np.zeros((len(s), 4), dtype=np.float64)
    ab = np.zeros(len(s), dtype=np.float64) if want_abs else None
    _check(lib().pk_ryser_f64_plan(_ptr(a), a.shape[0], int(cplx), PK_ALGO[algo], _ptr(s), _ptr(ln),
                                   len(s), int(devices), _ptr(out),
                                   _ptr(ab) if want_abs else None))
    return out, ab


def ryser_f64_batch(mats: np.ndarray, algo: str, devices: int = 1, want_abs: bool = False):
    """Full-range partials of B matrices; returns ([B,4] float64, [B] abs or None)."""
    cplx = np.iscomplexobj(mats)
    mats = np.ascontiguousarray(mats, dtype=np.complex128 if cplx else np.float64)
    B, n = mats.shape[0], mats.shape[1]
    out = np.zeros((B, 4), dtype=np.float64)
    ab = np.zeros(B, dtype=np.float64) if want_abs else None
    _check(lib().pk_ryser_f64_batch(_ptr(mats), B, n, int(cplx), PK_ALGO[algo], int(devices),
                                    _ptr(out), _ptr(ab) if want_abs else None))
    return out, ab


def ryser_modp(residues: np.ndarray, primes, algo: str, start: int, length: int,
               devices: int = 1) -> list:
    """Signed walk sums mod p for P residue matrices [P, n, n] (uint64)."""
    res = np.ascontiguousarray(residues, dtype=np.uint64)
    pr = np.ascontiguousarray(primes, dtype=np.uint64)
    P, n = res.shape[0], res.shape[1]
    out = np.zeros(P, dtype=np.uint64)
    _check(lib().pk_ryser_modp(_ptr(res), _ptr(pr), P, n, PK_ALGO[algo], int(start), int(length),
                               int(devices), _ptr(out)))
    return [int(x) for x in out]


def measure_peaks(device: int = 0) -> dict:
    buf = np.zeros(64, dtype=np.float64)
    k = lib().pk_measure_peaks(int(device), _ptr(buf), 64)
    if k < 0:
        _check(k)
    names = lib().pk_peak_names().decode().split(",")
    return {names[i]: {"ops_per_s": float(buf[3 * i]), "ops_per_clk_sm": float(buf[3 * i + 1]),
                       "sm_mhz": float(buf[3 * i + 2])} for i in range(k)}


def measure_mix_ceilings(device: int = 0) -> dict:
    """In-run ceilings of the walks' instruction mixes (csrc/pk_mix.cu)."""
    buf = np.zeros(48, dtype=np.float64)
    k = lib().pk_measure_mix_ceilings(int(device), _ptr(buf), 48)
    if k < 0:
        _check(k)
    names = lib().pk_mix_names().decode().split(",")
    return {names[i]: {"units_per_s": float(buf[3 * i]), "units_per_clk_sm": float(buf[3 * i + 1]),
                       "sm_mhz": float(buf[3 * i + 2])} for i in range(k)}


def kahan_fold(pairs: np.ndarray, is_complex: bool):
    """engine._run_plan's ordered combine (reference engine.py:240-245) in C:
    returns (sum, comp) of the per-block [s_re, s_im, c_re, c_im] rows."""
    pairs = np.ascontiguousarray(pairs, dtype=np.float64)
    out = np.zeros(4, dtype=np.float64)
    _check(lib().pk_kahan_fold(_ptr(pairs), pairs.shape[0], int(is_complex), _ptr(out)))
    if is_complex:
        return complex(out[0], out[1]), complex(out[2], out[3])
    return float(out[0]), float(out[2])


def measure_latencies(device: int = 0) -> dict:
    buf = np.zeros(16, dtype=np.float64)
    k = lib().pk_measure_latencies(int(device), _ptr(buf), 16)
    if k < 0:
        _check(k)
    names = lib().pk_latency_names().decode().split(",")
    return {names[i]: float(buf[i]) for i in range(k)}


class Job:
    """Device-resident walk (bench.py): inputs uploaded once, re-run many times."""

    def __init__(self, handle, kind: str, nres: int = 0):
        self._h = handle
        self.kind = kind
        self.nres = nres

    @classmethod
    def f64(cls, a: np.ndarray, algo: str, start: int, length: int, device: int = 0):
        cplx = np.iscomplexobj(a)
        a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
        h = _vp()
        _check(lib().pk_job_f64_create(int(device), _ptr(a), a.shape[0], int(cplx),
                                       PK_ALGO[algo], int(start), int(length), ctypes.byref(h)))
        return cls(h, "f64")

    @classmethod
    def modp(cls, residues: np.ndarray, primes, algo: str, start: int, length: int,
             device: int = 0):
        res = np.ascontiguousarray(residues, dtype=np.uint64)
        pr = np.ascontiguousarray(primes, dtype=np.uint64)
        h = _vp()
        _check(lib().pk_job_modp_create(int(device), _ptr(res), _ptr(pr), res.shape[0],
                                        res.shape[1], PK_ALGO[algo], int(start), int(length),
                                        ctypes.byref(h)))
        return cls(h, "modp", res.shape[0])

    def run(self, iters: int = 1, flush_bytes: int = 0):
        tot, walk = _dbl(0), _dbl(0)
        of = np.zeros(5, dtype=np.float64)
        orr = np.zeros(max(self.nres, 1), dtype=np.uint64)
        _check(lib().pk_job_run(self._h, int(iters), int(flush_bytes), ctypes.byref(tot),
                                ctypes.byref(walk), _ptr(of), _ptr(orr)))
        res = of.copy() if self.kind == "f64" else [int(x) for x in orr[: self.nres]]
        return tot.value, walk.value, res

    def info(self) -> dict:
        buf = np.zeros(8, dtype=np.int64)
        _check(lib().pk_job_info(self._h, _ptr(buf)))
        keys = ["k", "tiles", "grid", "ctas_per_sm", "regs", "local_bytes", "smem", "launches"]
        return {k: int(v) for k, v in zip(keys, buf)}

    GROUP_KINDS = ("reduced", "lazy", "hybrid", "hybrid_wide", "wide")

    def groups(self) -> list:
        """Per launch group of an F_p job: kind, primes (indices into the job's
        prime list), launch shape and the walk ms of the last run()."""
        desc = np.zeros((16, 6), dtype=np.int64)
        ms = np.zeros(16, dtype=np.float64)
        idx = np.zeros((16, 4), dtype=np.int64)
        g = lib().pk_job_groups(self._h, _ptr(desc), _ptr(ms), _ptr(idx), 16)
        if g < 0:
            _check(g)
        out = []
        for i in range(min(g, 16)):
            kind, P, regs, occ, grid, smem = (int(x) for x in desc[i])
            out.append({"kind": self.GROUP_KINDS[kind], "P": P, "regs": regs, "ctas_per_sm": occ,
                        "grid": grid, "smem": smem, "ms": float(ms[i]),
                        "prime_idx": [int(x) for x in idx[i] if x >= 0]})
        return out

    def close(self):
        if self._h:
            lib().pk_job_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
