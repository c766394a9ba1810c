// Per-block Gray walks with the reference's exact arithmetic.
//
// One thread walks one caller block [start, start + length) of the Gray index
// space exactly as the reference's numba kernels do, so the returned
// (sum, compensation) pair is bit-identical to kernels.ryser_partial /
// kernels.glynn_partial (reference kernels.py:33-226):
//   * no FMA contraction (explicit __dmul_rn / __dadd_rn / __dsub_rn),
//   * complex multiply (ac - bd) + (ad + bc)i with four separate products, as
//     numba lowers complex128 '*',
//   * the product starts from 1 (complex(1, 0)) and multiplies every state entry,
//   * flip direction from the current Gray code, Neumaier per component,
//   * Glynn's 2.0 * a promoted to complex(2, 0) * a as numba does.
// These kernels are the parity harness (pk_ryser_f64_blocks) and also walk the
// ragged head/tail of an unaligned range in the production path.
//
// The F_p block walker (any modulus 2 <= p < 2^62, reference kernels.py:229-344)
// returns the exact residue of the block; odd p use Montgomery-64, even p a
// 128-bit remainder.  Results are exact, so only the value has to agree.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pk_common.cuh"

namespace pk {

constexpr int kBlockMaxN = 64;
constexpr int kBlockThreads = 64;

struct C2 {
  double re, im;
};

__device__ __forceinline__ C2 cmul_ref(C2 x, C2 y) {
  const double ac = __dmul_rn(x.re, y.re), bd = __dmul_rn(x.im, y.im);
  const double ad = __dmul_rn(x.re, y.im), bc = __dmul_rn(x.im, y.re);
  return C2{__dsub_rn(ac, bd), __dadd_rn(ad, bc)};
}

__device__ __forceinline__ void neumaier_ref(double& s, double& c, double v) {
  const double t = __dadd_rn(s, v);
  if (fabs(s) >= fabs(v))
    c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), v));
  else
    c = __dadd_rn(c, __dadd_rn(__dsub_rn(v, t), s));
  s = t;
}

// steps in flight per thread (block_f64_kernel / block_modp_kernel skewed passes)
#ifndef PK_BLOCK_SKEW_REAL
#define PK_BLOCK_SKEW_REAL 4
#endif
#ifndef PK_BLOCK_SKEW_CPLX
#define PK_BLOCK_SKEW_CPLX 4
#endif
constexpr int block_skew(bool cplx, int nmax) {
  return !cplx ? PK_BLOCK_SKEW_REAL : nmax >= 64 ? 1 : nmax >= 48 ? 2 : PK_BLOCK_SKEW_CPLX;
}

__device__ __forceinline__ int ctz64(uint64_t x) { return __ffsll(static_cast<long long>(x)) - 1; }

// The state r[] is indexed only by unrolled loop counters below NMAX (guarded by
// i < n), so it lives in registers: NMAX is the smallest of 16 / 32 / 48 / 64 that
// holds n (block_nmax).  Skipped iterations do no arithmetic, so the operation
// sequence, and with it every bit, is the reference's for any NMAX >= n.
#define PK_FOR_ROWS(i) _Pragma("unroll") for (int i = 0; i < NMAX; ++i) if (i < n)

// out[blk * 4 + {0,1,2,3}] = (s_re, s_im, c_re, c_im); block blk walks matrix
// a + (blk / ppm) * mat_stride (ppm = nblocks, stride 0: one matrix)
template <bool CPLX, int ALGO, int NMAX>
__global__ void __launch_bounds__(kBlockThreads) block_f64_kernel(const double* __restrict__ a,
                                                                  int n,
                                                                  const uint64_t* __restrict__ starts,
                                                                  const uint64_t* __restrict__ lens,
                                                                  int nblocks, double* out,
                                                                  double* abs_out, int ppm,
                                                                  size_t mat_stride) {
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;
  if (blk >= nblocks) return;
  a += static_cast<size_t>(blk / ppm) * mat_stride;  // ppm blocks per matrix (batched pieces)
  C2 r[NMAX];
  double abs_acc = 0.0;
  auto A = [&](int i, int j) -> C2 {
    if constexpr (CPLX) return C2{a[2 * (i * n + j)], a[2 * (i * n + j) + 1]};
    return C2{a[i * n + j], 0.0};
  };
  const uint64_t start = starts[blk], length = lens[blk];
  uint64_t g = start ^ (start >> 1);
  int pop = 0;
  if constexpr (ALGO == 0) {
    PK_FOR_ROWS(i) r[i] = C2{0.0, 0.0};
    for (int j = 0; j < n; ++j) {
      if ((g >> j) & 1) {
        ++pop;
        PK_FOR_ROWS(i) {
          const C2 x = A(i, j);
          r[i].re = __dadd_rn(r[i].re, x.re);
          if constexpr (CPLX) r[i].im = __dadd_rn(r[i].im, x.im);
        }
      }
    }
  } else {
    PK_FOR_ROWS(j) r[j] = A(0, j);
    for (int i = 0; i < n - 1; ++i) {
      const bool on = (g >> i) & 1;
      pop += on;
      PK_FOR_ROWS(j) {
        const C2 x = A(i + 1, j);
        if (on) {
          r[j].re = __dsub_rn(r[j].re, x.re);
          if constexpr (CPLX) r[j].im = __dsub_rn(r[j].im, x.im);
        } else {
          r[j].re = __dadd_rn(r[j].re, x.re);
          if constexpr (CPLX) r[j].im = __dadd_rn(r[j].im, x.im);
        }
      }
    }
  }
  int neg = ALGO == 0 ? ((n - pop) & 1) : (pop & 1);
  double s_re = 0.0, c_re = 0.0, s_im = 0.0, c_im = 0.0;
  uint64_t idx = start;
  uint64_t step = 0;
  // KS steps per pass, skewed: at row i, chain k multiplies row i of step + k and
  // then moves that row to step + k + 1, which is exactly what chain k + 1 reads
  // next.  Each step's product and update sequence is unchanged (bit-identical),
  // but KS independent product chains are in flight instead of one.
  constexpr int KS = block_skew(CPLX, NMAX);
  for (; KS > 1 && step + KS < length; step += KS) {
    int bk[KS];
    bool sk[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      bk[k] = ctz64(++idx);
      sk[k] = (g >> bk[k]) & 1;
      g ^= 1ull << bk[k];
    }
    C2 pr[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) pr[k] = C2{1.0, 0.0};
    PK_FOR_ROWS(i) {
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        if constexpr (CPLX)
          pr[k] = cmul_ref(pr[k], r[i]);
        else
          pr[k].re = __dmul_rn(pr[k].re, r[i].re);
        if constexpr (ALGO == 0) {
          const C2 x = A(i, bk[k]);
          if (sk[k]) {
            r[i].re = __dsub_rn(r[i].re, x.re);
            if constexpr (CPLX) r[i].im = __dsub_rn(r[i].im, x.im);
          } else {
            r[i].re = __dadd_rn(r[i].re, x.re);
            if constexpr (CPLX) r[i].im = __dadd_rn(r[i].im, x.im);
          }
        } else {
          const C2 x = A(bk[k] + 1, i);
          C2 two;
          if constexpr (CPLX)
            two = cmul_ref(C2{2.0, 0.0}, x);
          else
            two = C2{__dmul_rn(2.0, x.re), 0.0};
          if (sk[k]) {
            r[i].re = __dadd_rn(r[i].re, two.re);
            if constexpr (CPLX) r[i].im = __dadd_rn(r[i].im, two.im);
          } else {
            r[i].re = __dsub_rn(r[i].re, two.re);
            if constexpr (CPLX) r[i].im = __dsub_rn(r[i].im, two.im);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const double v_re = neg ? -pr[k].re : pr[k].re;
      const double v_im = CPLX ? (neg ? -pr[k].im : pr[k].im) : 0.0;
      neumaier_ref(s_re, c_re, v_re);
      if constexpr (CPLX) neumaier_ref(s_im, c_im, v_im);
      if (abs_out) abs_acc += fabs(v_re) + fabs(v_im);
      neg ^= 1;
    }
  }
  for (; step < length; ++step) {
    double v_re, v_im = 0.0;
    if constexpr (CPLX) {
      C2 prod{1.0, 0.0};
      PK_FOR_ROWS(i) prod = cmul_ref(prod, r[i]);
      v_re = neg ? -prod.re : prod.re;
      v_im = neg ? -prod.im : prod.im;
    } else {
      double prod = 1.0;
      PK_FOR_ROWS(i) prod = __dmul_rn(prod, r[i].re);
      v_re = neg ? -prod : prod;
    }
    neumaier_ref(s_re, c_re, v_re);
    if constexpr (CPLX) neumaier_ref(s_im, c_im, v_im);
    if (abs_out) abs_acc += fabs(v_re) + fabs(v_im);
    if (step + 1 < length) {
      ++idx;
      const int b = ctz64(idx);
      const bool set = (g >> b) & 1;
      if constexpr (ALGO == 0) {
        PK_FOR_ROWS(i) {
          const C2 x = A(i, b);
          if (set) {
            r[i].re = __dsub_rn(r[i].re, x.re);
            if constexpr (CPLX) r[i].im = __dsub_rn(r[i].im, x.im);
          } else {
            r[i].re = __dadd_rn(r[i].re, x.re);
            if constexpr (CPLX) r[i].im = __dadd_rn(r[i].im, x.im);
          }
        }
      } else {
        PK_FOR_ROWS(j) {
          const C2 x = A(b + 1, j);
          C2 two;
          if constexpr (CPLX)
            two = cmul_ref(C2{2.0, 0.0}, x);  // numba: float * complex -> complex(2, 0) * x
          else
            two = C2{__dmul_rn(2.0, x.re), 0.0};
          if (set) {
            r[j].re = __dadd_rn(r[j].re, two.re);
            if constexpr (CPLX) r[j].im = __dadd_rn(r[j].im, two.im);
          } else {
            r[j].re = __dsub_rn(r[j].re, two.re);
            if constexpr (CPLX) r[j].im = __dsub_rn(r[j].im, two.im);
          }
        }
      }
      g ^= 1ull << b;
      neg ^= 1;
    }
  }
  out[4 * blk + 0] = s_re;
  out[4 * blk + 1] = s_im;
  out[4 * blk + 2] = c_re;
  out[4 * blk + 3] = c_im;
  if (abs_out) abs_out[blk] = abs_acc;
}

// smallest register-state bound that holds n (n <= kBlockMaxN)
inline int block_nmax(int n) { return n <= 16 ? 16 : n <= 32 ? 32 : n <= 48 ? 48 : 64; }

// ---------------------------------------------------------------------------
// F_p blocks, any modulus 2 <= p < 2^62.

struct ModArith {
  uint64_t p, mneg;
  bool odd;
  __device__ __forceinline__ uint64_t add(uint64_t x, uint64_t y) const {
    const uint64_t v = x + y;  // < 2^63
    return v >= p ? v - p : v;
  }
  __device__ __forceinline__ uint64_t neg(uint64_t x) const { return x == 0 ? 0 : p - x; }
  // odd p: Montgomery product x*y*2^-64; even p: plain x*y mod p
  __device__ __forceinline__ uint64_t mul(uint64_t x, uint64_t y) const {
    if (odd) {
      const uint64_t lo = x * y, hi = __umul64hi(x, y);
      const uint64_t mm = lo * mneg;
      const uint64_t u = hi + __umul64hi(mm, p) + (lo != 0 ? 1ull : 0ull);
      return u >= p ? u - p : u;
    }
    const unsigned __int128 t = static_cast<unsigned __int128>(x) * y;
    return static_cast<uint64_t>(t % p);
  }
};

// out[blk] = sum over the block of sign * prod(state) with the product in
// Montgomery scale 2^(-64 (n-1)) for odd p (the host multiplies by 2^(64(n-1))),
// and plain for even p.  Glynn's 2^(1-n) is applied by the caller, as in the
// reference engine (engine.py:252-258).
template <int ALGO, int NMAX>
__global__ void __launch_bounds__(kBlockThreads) block_modp_kernel(const uint64_t* __restrict__ a,
                                                                   int n, uint64_t p,
                                                                   const uint64_t* __restrict__ starts,
                                                                   const uint64_t* __restrict__ lens,
                                                                   int nblocks, uint64_t* out) {
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;
  if (blk >= nblocks) return;
  ModArith ar{p, (p & 1) ? mont_neg_inv64(p) : 0ull, (p & 1) != 0};
  uint64_t r[NMAX];
  const uint64_t start = starts[blk], length = lens[blk];
  uint64_t g = start ^ (start >> 1);
  int pop = 0;
  if constexpr (ALGO == 0) {
    PK_FOR_ROWS(i) r[i] = 0;
    for (int j = 0; j < n; ++j)
      if ((g >> j) & 1) {
        ++pop;
        PK_FOR_ROWS(i) r[i] = ar.add(r[i], a[i * n + j]);
      }
  } else {
    PK_FOR_ROWS(j) r[j] = a[j];
    for (int i = 0; i < n - 1; ++i) {
      const bool on = (g >> i) & 1;
      pop += on;
      PK_FOR_ROWS(j) {
        const uint64_t x = a[(i + 1) * n + j];
        r[j] = ar.add(r[j], on ? ar.neg(x) : x);
      }
    }
  }
  int neg = ALGO == 0 ? ((n - pop) & 1) : (pop & 1);
  uint64_t acc = 0;
  uint64_t idx = start;
  uint64_t step = 0;
  constexpr int KS = block_skew(false, NMAX);  // skewed passes, as in block_f64_kernel
  for (; step + KS < length; step += KS) {
    int bk[KS];
    bool sk[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      bk[k] = ctz64(++idx);
      sk[k] = (g >> bk[k]) & 1;
      g ^= 1ull << bk[k];
    }
    uint64_t pr[KS];
    PK_FOR_ROWS(i) {
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        pr[k] = i == 0 ? r[0] : ar.mul(pr[k], r[i]);
        if constexpr (ALGO == 0) {
          const uint64_t x = a[i * n + bk[k]];
          r[i] = ar.add(r[i], sk[k] ? ar.neg(x) : x);
        } else {
          const uint64_t x = a[(bk[k] + 1) * n + i];
          const uint64_t two = ar.add(x, x);
          r[i] = ar.add(r[i], sk[k] ? two : ar.neg(two));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      acc = ar.add(acc, neg ? ar.neg(pr[k]) : pr[k]);
      neg ^= 1;
    }
  }
  for (; step < length; ++step) {
    uint64_t prod = r[0];
    _Pragma("unroll") for (int i = 1; i < NMAX; ++i) if (i < n) prod = ar.mul(prod, r[i]);
    acc = ar.add(acc, neg ? ar.neg(prod) : prod);
    if (step + 1 < length) {
      ++idx;
      const int b = ctz64(idx);
      const bool set = (g >> b) & 1;
      if constexpr (ALGO == 0) {
        PK_FOR_ROWS(i) {
          const uint64_t x = a[i * n + b];
          r[i] = ar.add(r[i], set ? ar.neg(x) : x);
        }
      } else {
        PK_FOR_ROWS(j) {
          const uint64_t x = a[(b + 1) * n + j];
          const uint64_t two = ar.add(x, x);
          r[j] = ar.add(r[j], set ? two : ar.neg(two));
        }
      }
      g ^= 1ull << b;
      neg ^= 1;
    }
  }
  out[blk] = acc;
}

#undef PK_FOR_ROWS

}  // namespace pk
