"""Random-matrix ensembles and the batched permanent sampler.

Sampling is kept bit-identical to the reference (reference
pkg/src/permkit/ensembles.py:18-158): sample i of (kind, n, seed) comes from
PCG64(SeedSequence((seed, i))) through Marsaglia-polar normals, so any
worker/device count reproduces the same matrices.  The permanents, which the
reference evaluates one per thread-pool task (ensembles.py:149-157), are
evaluated here in batches on the GPU (``engine.perm_batch``): matrices are
generated on host threads in chunks while the previous chunk's walk runs.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .engine import perm_batch
from .matrices import qr_decompose

ENSEMBLES = ("haar-u", "haar-o", "gue", "goe", "ginibre-c", "ginibre-r")


@dataclass(frozen=True)
class EnsembleSpec:
    kind: str
    n: int
    count: int
    seed: int

    def __post_init__(self):
        if self.kind not in ENSEMBLES:
            raise ValueError(f"unknown ensemble {self.kind!r}")
        if self.n < 1 or self.count < 1:
            raise ValueError("n and count must be >= 1")


class RngStream:
    """Counter-keyed stream: PCG64 seeded by SeedSequence((seed, stream))."""

    def __init__(self, seed: int, stream: int):
        self.seed, self.stream = int(seed), int(stream)
        self._rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence((self.seed,
                                                                                 self.stream))))

    def uniforms(self, count: int) -> np.ndarray:
        return self._rng.random(count)

    def normals(self, count: int) -> np.ndarray:
        """Polar-method normals; whole (u, v) pairs are consumed, a trailing odd one dropped.

        Each round draws max(8, 1.35 * pairs_missing + 4) candidate pairs
        (u's first, then v's), keeps those with 0 < u^2 + v^2 < 1 in order and
        maps each to (u f, v f), f = sqrt(-2 ln s / s).
        """
        pairs = (count + 1) // 2
        out = np.empty(2 * pairs)
        filled = 0  # pairs written
        while filled < pairs:
            missing = pairs - filled
            draws = max(8, int(missing * 1.35) + 4)
            u = 2.0 * self._rng.random(draws) - 1.0
            v = 2.0 * self._rng.random(draws) - 1.0
            s = u * u + v * v
            keep = (s > 0.0) & (s < 1.0)
            u, v, s = u[keep][:missing], v[keep][:missing], s[keep][:missing]
            f = np.sqrt(-2.0 * np.log(s) / s)
            k = len(s)
            out[2 * filled:2 * (filled + k):2] = u * f
            out[2 * filled + 1:2 * (filled + k):2] = v * f
            filled += k
        return out[:count]


def gaussian_draw(stream: RngStream) -> float:
    return float(stream.normals(1)[0])


def _cnormals(stream: RngStream, count: int) -> np.ndarray:
    z = stream.normals(2 * count)
    return (z[0::2] + 1j * z[1::2]) / np.sqrt(2.0)


def _haar_fix(q, d_raw, unitary: bool):
    if unitary:
        d = np.where(d_raw == 0, 1.0, d_raw / np.abs(d_raw))
    else:
        d = np.sign(d_raw)
        d = np.where(d == 0, 1.0, d)
    return np.ascontiguousarray(q * d[None, :])


def sample_matrix(kind: str, n: int, seed: int, index: int) -> np.ndarray:
    """Matrix ``index`` of the (kind, n, seed) run."""
    st = RngStream(seed, index)
    if kind == "ginibre-c":
        return _cnormals(st, n * n).reshape(n, n)
    if kind == "ginibre-r":
        return st.normals(n * n).reshape(n, n)
    if kind == "gue":
        g = _cnormals(st, n * n).reshape(n, n)
        return (g + g.conj().T) / 2.0
    if kind == "goe":
        g = st.normals(n * n).reshape(n, n)
        return (g + g.T) / 2.0
    if kind == "haar-u":
        q, r = qr_decompose(_cnormals(st, n * n).reshape(n, n))
        return _haar_fix(q, np.diagonal(r).copy(), True)
    if kind == "haar-o":
        q, r = np.linalg.qr(st.normals(n * n).reshape(n, n))
        return _haar_fix(q, np.diagonal(r), False)
    raise ValueError(f"unknown ensemble {kind!r}")


def _typed_sampler(kinds, message):
    def sampler(spec: EnsembleSpec, index: int = 0) -> np.ndarray:
        if spec.kind not in kinds:
            raise ValueError(message)
        return sample_matrix(spec.kind, spec.n, spec.seed, index)
    return sampler


sample_ginibre = _typed_sampler(("ginibre-c", "ginibre-r"), "spec is not a Ginibre ensemble")
sample_gue = _typed_sampler(("gue",), "spec is not GUE")
sample_goe = _typed_sampler(("goe",), "spec is not GOE")
sample_haar_unitary = _typed_sampler(("haar-u",), "spec is not the unitary Haar ensemble")
sample_haar_orthogonal = _typed_sampler(("haar-o",), "spec is not the orthogonal Haar ensemble")


def sample_batch(spec: EnsembleSpec, start: int, stop: int, threads: int | None = None):
    """Matrices [start, stop) of a run as one [k, n, n] array (host threads)."""
    idx = range(start, stop)
    threads = threads or min(32, os.cpu_count() or 1)
    if threads > 1 and len(idx) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            mats = list(pool.map(lambda i: sample_matrix(spec.kind, spec.n, spec.seed, i), idx))
    else:
        mats = [sample_matrix(spec.kind, spec.n, spec.seed, i) for i in idx]
    return np.stack(mats)


def sample_permanents(spec: EnsembleSpec, method: str = "ryser", threads: int = 1,
                      devices: int | None = None, chunk: int | None = None) -> np.ndarray:
    """Permanents of ``spec.count`` fresh ensemble matrices, complex128 [count].

    Host generation of chunk c+1 overlaps the GPU walk of chunk c.  The
    output does not depend on threads, devices or chunking.
    """
    chunk = chunk or max(1, min(spec.count, 4096))
    bounds = [(s, min(spec.count, s + chunk)) for s in range(0, spec.count, chunk)]
    out = np.empty(spec.count, dtype=np.complex128)
    gen_threads = max(threads, min(32, os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=1) as pre:
        fut = pre.submit(sample_batch, spec, *bounds[0], gen_threads)
        for k, (s, e) in enumerate(bounds):
            mats = fut.result()
            if k + 1 < len(bounds):
                fut = pre.submit(sample_batch, spec, *bounds[k + 1], gen_threads)
            out[s:e] = perm_batch(mats, method=method, devices=devices)
    return out
