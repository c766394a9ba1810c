// Production Gray-code walk kernels (fp64 real/complex and F_p Montgomery-32).
//
// One kernel skeleton serves Ryser and Glynn.  Both expansions walk a Gray
// index space [0, 2^m) and keep an n-vector state
//     state(S) = base + sum_{b in S} w_b,     term(S) = sgn0 * (-1)^|S| * prod_i state_i(S)
//   Ryser (reference kernels.py:33-123, 250-290):  m = n,   base = 0,          w_b = a[:, b],
//                                                  sgn0 = (-1)^n
//   Glynn (reference kernels.py:126-226, 293-344): m = n-1, base = sum_i a[i,:], w_b = -2 a[b+1,:],
//                                                  sgn0 = +1, caller scales by 2^(1-n)
// so the walk matrix W = [w_0 .. w_{m-1}] and base are built once in shared
// memory when a matrix is staged, and the hot loop is identical.
//
// Work decomposition (B200-first):
//   segment = 2^k consecutive Gray indices walked by ONE lane; segments are
//             aligned, so at step s of every lane the flip column is ctz(s)
//             (warp-uniform => shared-memory broadcast, no divergence) and the
//             flip direction is bit ctz(s)+1 of s, except at ctz(s) = k-1
//             where it is bit 0 of the segment index (per lane).
//   product = a balanced binary tree over the n state entries (n-1 multiplies,
//             depth log2 n): the FP64 complex link (DMUL->DFMA) is 16 cycles
//             and a Montgomery REDC link 28 cycles on B200, so a serial chain
//             is latency bound at 2-3 resident warps per scheduler.
//   tile    = 32 consecutive segments = one warp; the warp reduces its lanes
//             with a fixed shuffle tree -> one partial per tile.
//   Tiles are spread over a persistent grid (grid-stride over warps); tile
//   partials are reduced by reduce_tiles_kernel in a fixed, device-count
//   independent tree (fp64) or summed mod p (F_p, exact, order-free).
// The start state of a segment is rebuilt in O((m-k) n) from gray(start),
// mirroring gray.block_start_state (reference gray.py:88-114).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "pk_common.cuh"

#ifndef PK_MINCTA_T
#define PK_MINCTA_T 64
#endif
// Column 0 in the kernel parameter: read element by element (0, default) or as
// 16-byte double2 vectors from an alignas(16) field (1).  The element-wise form
// keeps round 1's parameter layout, which measured 1.5 % faster on the complex
// n = 32 walk (57.45 vs 58.4 ms, profiles/r2_col0_layout.txt) -- a scheduling
// effect of the layout, since both read column 0 as LDCU.128 -- and needs no
// cast of the parameter to double2 (no misaligned vector access).
#ifndef PK_COL0_ALIGN
#define PK_COL0_ALIGN 0
#endif
// PK_PAIR4 (experiment, off): two step pairs per compensated add (one Neumaier
// step per four terms).  The loop body then holds two odd steps; their column-0
// reads come from two parameter copies (WalkArgs::col0, col0b) so both stay
// uniform-register operands.  Measured 57.22 vs 57.37 ms complex, 20.01 vs
// 20.30 ms real at n = 32 (profiles/r2_pair4.txt), but the batched
// per-warp-slot kernels spill with the four-step body, and a pair-per-step
// batch would no longer match a single call bit for bit: not adopted.
#ifndef PK_PAIR4
#define PK_PAIR4 0
#endif
namespace pk {

constexpr int kWalkThreads = 128;  // 4 warps per CTA
constexpr int kWalkWarps = kWalkThreads / 32;
constexpr int kTileBits = 5;       // 32 segments (lanes) per warp-tile

// Per-launch modulus constants (F_p kernels).  Read through a pointer into the
// __grid_constant__ kernel parameter, they compile to uniform-register / constant
// operands of IMAD / IMAD.HI / DFMA, costing no vector-register reads.
struct ModConsts {
  uint32_t p[4], mneg[4], kneg[4];  // Montgomery primes, -p^-1 mod 2^32, REDC output bound
  double fp[2], fpinv[2];           // fp64 primes (hybrid kernel) and 1/p
  uint64_t p64[2], pinv64[2];       // wide moduli 2^31 <= p < 2^62 and p^-1 mod 2^64
};

struct WalkArgs {
  const void* a;         // B matrices, row-major n x n (real f64, complex f64 interleaved, or
                         // P x n x n uint32 residues for F_p)
  int B;                 // matrices (F_p: prime groups)
  int n;                 // state length
  int m;                 // Gray bits: n (Ryser) or n-1 (Glynn)
  int algo;              // 0 Ryser, 1 Glynn
  int k;                 // segment bits (segment = 2^k indices), k >= 1
  int per_warp_slot;     // 1: every warp stages its own matrix (batched mode)
  uint64_t tile0;        // first global tile index of the launch (same for every matrix)
  uint64_t tiles;        // tiles per matrix in this launch
  uint64_t segs_total;   // 2^(m-k): segments per matrix (lanes beyond are idle)
  double* partials;      // fp64: [B][tiles][5] = (s_re, c_re, s_im, c_im, abs)
  unsigned long long* modp_out;  // F_p: [B][P] raw sums (< 2^64, reduced on host)
  const uint32_t* primes;        // F_p: [B][P]
  int want_abs;          // fp64: accumulate sum |term| (parity tolerance)
  ModConsts mc;          // F_p: constants of the (single) prime group of the launch
  // fp64, one matrix per launch (C0P kernels): walk column 0 (n values, complex
  // interleaved), flipped on every odd step.  Read through the __grid_constant__
  // parameter it compiles to uniform-register DFMA operands (LDCU): no shared
  // load and no register-file read for half of all steps.
  // (F_p kernels keep column 0 in shared memory: with parameter operands the
  // lazy walk measured 8-10 % slower, profiles/r1_modp_rates_c0.json.)
#if PK_COL0_ALIGN
  alignas(16) double col0[2 * 48];  // read as double2 by the complex walker
#else
  double col0[2 * 48];  // read element by element (F64Walker::step_c0)
#endif
#if PK_PAIR4
  double col0b[2 * 48];  // a second copy of col0 (PK_PAIR4)
#endif
};
#if PK_COL0_ALIGN
static_assert(offsetof(WalkArgs, col0) % 16 == 0, "WalkArgs::col0 must be 16-byte aligned");
#endif

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Row stride of one column in shared memory, a multiple of the 16-byte vector.
__host__ __device__ constexpr int col_stride(int n, int elem_bytes) {
  const int align = 16 / elem_bytes;
  return (n + align - 1) / align * align;
}

// Resident CTAs per SM the launch bounds ask for: 3 while the register-resident
// state is small, 2 when it is large (spilling the state costs more than the
// lost occupancy: the product trees give plenty of ILP per warp).
__host__ __device__ constexpr int min_ctas(int state_regs) { return state_regs > PK_MINCTA_T ? 2 : 3; }

// Gray-step bookkeeping shared by the fp64 and F_p walkers.
struct StepPlan {
  // direction (true = remove the column) of the even step e >= 2
  __device__ __forceinline__ static bool minus_even(uint32_t e, int k, bool lane_minus) {
    const int b = __ffs(e) - 1;
    return (b == k - 1) ? lane_minus : ((e >> (b + 1)) & 1);
  }
  // direction of the odd step o (column 0)
  __device__ __forceinline__ static bool minus_odd(uint32_t o, int k, bool lane_minus) {
    return (k == 1) ? lane_minus : ((o >> 1) & 1);
  }
};

// ---------------------------------------------------------------------------
// fp64

template <bool CPLX>
struct F64T;
template <>
struct F64T<false> {
  using T = double;
  static constexpr int kBytes = 8;
  __device__ static T zero() { return 0.0; }
  __device__ static T load(const double* a, int idx) { return a[idx]; }
};
template <>
struct F64T<true> {
  using T = double2;
  static constexpr int kBytes = 16;
  __device__ static T zero() { return make_double2(0.0, 0.0); }
  __device__ static T load(const double* a, int idx) {
    return make_double2(a[2 * idx], a[2 * idx + 1]);
  }
};

__device__ __forceinline__ void fma_upd(double& r, double sg, double c) { r = fma(sg, c, r); }
__device__ __forceinline__ void fma_upd(double2& r, double sg, double2 c) {
  r.x = fma(sg, c.x, r.x);
  r.y = fma(sg, c.y, r.y);
}
__device__ __forceinline__ void mul_acc(double& p, double v) { p *= v; }
__device__ __forceinline__ void mul_acc(double2& p, double2 v) {
  const double nr = fma(p.x, v.x, -(p.y * v.y));
  p.y = fma(p.x, v.y, p.y * v.x);
  p.x = nr;
}
__device__ __forceinline__ double2 sub2(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double sub2(double a, double b) { return a - b; }

// Neumaier step in the reference's form (kernels.py:56-67): t = s + v;
// c += (big - t) + small.
__device__ __forceinline__ void neumaier(double& s, double& c, double v) {
  const double t = s + v;
  const bool sb = fabs(s) >= fabs(v);
  const double big = sb ? s : v;
  const double small = sb ? v : s;
  c += (big - t) + small;
  s = t;
}

// Stage one matrix in walk form: base[NS] then W[m][NS] (NS = padded n).
// Shared layout: base[NS] | W[m][NS] (| Wm[m][NS] = -W when MINUS: the
// single-matrix kernels flip even-step columns with a two-operand DADD).
template <int N, bool CPLX, bool MINUS = false>
__device__ void stage_f64(typename F64T<CPLX>::T* sm, const double* a, int m, int algo, int tid,
                          int nthreads) {
  using F = F64T<CPLX>;
  using T = typename F::T;
  constexpr int NS = col_stride(N, F::kBytes);
  T* base = sm;
  T* W = sm + NS;
  for (int idx = tid; idx < (m + 1) * NS; idx += nthreads) {
    const int i = idx % NS;
    const int b = idx / NS - 1;  // -1: base
    T v = F::zero();
    if (i >= N) {
      // padding: never read
    } else if (b < 0) {
      if (algo == 1) {  // Glynn base: column sums sum_r a[r][i]
        v = F::load(a, i);
        for (int r = 1; r < N; ++r) {
          const T x = F::load(a, r * N + i);
          if constexpr (CPLX) {
            v.x += x.x;
            v.y += x.y;
          } else {
            v += x;
          }
        }
      }
    } else if (algo == 0) {
      v = F::load(a, i * N + b);  // Ryser: W[b][i] = a[i][b]
    } else {
      v = F::load(a, (b + 1) * N + i);  // Glynn: W[b][i] = -2 a[b+1][i]
      if constexpr (CPLX) {
        v.x *= -2.0;
        v.y *= -2.0;
      } else {
        v *= -2.0;
      }
    }
    (b < 0 ? base : W + b * NS)[i] = v;
    if (MINUS && b >= 0) {
      T nv = v;
      if constexpr (CPLX) {
        nv.x = -v.x;
        nv.y = -v.y;
      } else {
        nv = -v;
      }
      W[(m + b) * NS + i] = nv;
    }
  }
}

// C0P: column 0 comes from the kernel parameter (WalkArgs::col0) instead of
// shared memory; measured +6 % (complex) / +9 % (real) at n = 32
// (profiles/r1_walk_experiments.txt).  Batched launches (a matrix per warp)
// keep it in shared memory.
template <int N, bool CPLX, bool C0P>
struct F64Walker {
  using F = F64T<CPLX>;
  using T = typename F::T;
  static constexpr int NS = col_stride(N, F::kBytes);

  T r[N];
  double s_re, c_re, s_im, c_im, abs_acc;
  bool want_abs;
  const T* c0;  // C0P: column 0 in the __grid_constant__ parameter
  const double* c0d;  // the same, as doubles (PK_COL0_ALIGN = 0)
  const double* c0d2;  // PK_PAIR4: the second copy (WalkArgs::col0b)
  // shared minus copies of the walk columns (DADD flips): single-matrix kernels
  // only; in the batched kernels (a slot per warp) they measured -1 to -15 %
  static constexpr bool kMinus = C0P;

  // Product of the state as a binary tree evaluated depth-first (a binary
  // counter over the leaves): the same N - 1 multiplies as a chain, depth
  // ~log2 N, and at most log2 N + 1 partial products live at once.
  __device__ __forceinline__ T tree() const {
    constexpr int LOG = 7;
    T st[LOG];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      T v = r[j];
      int l = 0;
#pragma unroll
      for (; l < LOG && ((j >> l) & 1); ++l) {
        mul_acc(st[l], v);
        v = st[l];
      }
      st[l] = v;
    }
    // leftover complete subtrees: one per set bit of N, lowest first
    T acc = r[0];
    bool have = false;
#pragma unroll
    for (int l = 0; l < LOG; ++l) {
      if ((N >> l) & 1) {
        if (have) {
          mul_acc(acc, st[l]);
        } else {
          acc = st[l];
          have = true;
        }
      }
    }
    return acc;
  }

  // flip one column with direction sg and return the new term's product
  __device__ __forceinline__ T step(const T* __restrict__ col, double sg) {
    update(col, sg);
    return tree();
  }
  // column 0 from the kernel parameter, read element by element
  __device__ __forceinline__ T step_c0(const double* __restrict__ c, double sg) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if constexpr (CPLX)
        fma_upd(r[j], sg, make_double2(c[2 * j], c[2 * j + 1]));
      else
        fma_upd(r[j], sg, c[j]);
    }
    return tree();
  }

  __device__ __forceinline__ void update(const T* __restrict__ col, double sg) {
    if constexpr (CPLX) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
#ifdef PK_EXP_NOLDS  // micro-experiments only: column from registers
        fma_upd(r[j], sg, make_double2(1e-3 * j, 1e-3));
#else
        fma_upd(r[j], sg, col[j]);
#endif
      }
    } else {
#pragma unroll
      for (int j = 0; j + 2 <= N; j += 2) {  // two rows per 16-byte load
        const double2 c2 = *reinterpret_cast<const double2*>(col + j);
        fma_upd(r[j], sg, c2.x);
        fma_upd(r[j + 1], sg, c2.y);
      }
      if constexpr (N & 1) fma_upd(r[N - 1], sg, col[N - 1]);
    }
  }

  // Terms of a step pair (even e, odd e+1) carry opposite signs: their
  // difference is formed in plain fp64 (one rounding, <= u (|t_e| + |t_o|))
  // and compensated-added once, halving the Neumaier work.
  // PK_BLOCK_SUM (experiment): the pair differences of kBlockPairs consecutive
  // pairs are summed plainly (error <= kBlockPairs u sum |t|, inside the n u S
  // gate for kBlockPairs <= n) and compensated-added once per block
#ifndef PK_BLOCK_SUM
#define PK_BLOCK_SUM 0
#endif
  static constexpr uint32_t kBlockPairs = 8;
  T pend;
  __device__ __forceinline__ void add_pair_blk(T pe, T po, bool flush) {
    if constexpr (!PK_BLOCK_SUM) {
      add_pair(pe, po);
      return;
    }
    const T d = sub2(pe, po);
    if constexpr (CPLX) {
      pend.x += d.x;
      pend.y += d.y;
      if (want_abs) abs_acc += (fabs(pe.x) + fabs(pe.y)) + (fabs(po.x) + fabs(po.y));
      if (flush) {
        neumaier(s_re, c_re, pend.x);
        neumaier(s_im, c_im, pend.y);
        pend = F::zero();
      }
    } else {
      pend += d;
      if (want_abs) abs_acc += fabs(pe) + fabs(po);
      if (flush) {
        neumaier(s_re, c_re, pend);
        pend = F::zero();
      }
    }
  }

  __device__ __forceinline__ void add_pair(T pe, T po) {
    const T d = sub2(pe, po);
#ifdef PK_EXP_NOKAHAN  // micro-experiments only (tools/micro): plain sums
    if constexpr (CPLX) {
      s_re += d.x;
      s_im += d.y;
    } else {
      s_re += d;
    }
    return;
#endif
    if constexpr (CPLX) {
      neumaier(s_re, c_re, d.x);
      neumaier(s_im, c_im, d.y);
      if (want_abs) abs_acc += (fabs(pe.x) + fabs(pe.y)) + (fabs(po.x) + fabs(po.y));
    } else {
      neumaier(s_re, c_re, d);
      if (want_abs) abs_acc += fabs(pe) + fabs(po);
    }
  }

  __device__ __forceinline__ void add_quad(T pe, T po, T qe, T qo) {
    const T d = sub2(pe, po);
    const T f = sub2(qe, qo);
    if constexpr (CPLX) {
      neumaier(s_re, c_re, d.x + f.x);
      neumaier(s_im, c_im, d.y + f.y);
      if (want_abs)
        abs_acc += ((fabs(pe.x) + fabs(pe.y)) + (fabs(po.x) + fabs(po.y))) +
                   ((fabs(qe.x) + fabs(qe.y)) + (fabs(qo.x) + fabs(qo.y)));
    } else {
      neumaier(s_re, c_re, d + f);
      if (want_abs) abs_acc += (fabs(pe) + fabs(po)) + (fabs(qe) + fabs(qo));
    }
  }

  // PK_PAIR4 only where the four-step body fits the register file without
  // spilling (single-matrix kernels, complex n <= 37, real n <= 63)
  static constexpr bool kPair4 = PK_PAIR4 && C0P && (CPLX ? N <= 37 : N <= 63);

  static constexpr int kSubBits = 12;
  __device__ __forceinline__ void walk(const T* __restrict__ base, const T* __restrict__ W, int m,
                                       int k, uint64_t seg) {
    s_re = c_re = s_im = c_im = abs_acc = 0.0;
    const int ks = min(k, kSubBits);
    const uint32_t nsub = 1u << (k - ks);
    for (uint32_t i = 0; i < nsub; ++i) walk_sub(base, W, m, ks, (seg << (k - ks)) | i);
  }

  // Walk segment `seg` (2^k indices starting at seg << k).
  __device__ __forceinline__ void walk_sub(const T* __restrict__ base, const T* __restrict__ W,
                                           int m, int k, uint64_t seg) {
    const uint64_t start = seg << k;
    const uint64_t g = start ^ (start >> 1);
    const T* bp = base + (start >> 63) * NS;  // not hoisted out of the sub-segment loop
#pragma unroll
    for (int j = 0; j < N; ++j) r[j] = bp[j];
    for (int b = k - 1; b < m; ++b) {  // start state: columns set in gray(start)
      const double on = ((g >> b) & 1) ? 1.0 : 0.0;
      const T* col = W + b * NS;
#pragma unroll
      for (int j = 0; j < N; ++j) fma_upd(r[j], on, col[j]);
    }
    const uint32_t L = 1u << k;
    const bool lane_minus = seg & 1;
    {  // steps 0 (no flip) and 1
      const T pe = tree();
      // (start >> 63) is always 0: keeps column 0 from being hoisted out of the
      // sub-segment loop into registers
      const bool mo = StepPlan::minus_odd(1, k, lane_minus);
      const T po = kMinus ? step((mo ? W + m * NS : W) + (start >> 63) * NS, 1.0)
                          : step(W + (start >> 63) * NS, mo ? -1.0 : 1.0);
      pend = F::zero();
      add_pair_blk(pe, po, L == 2);
    }
    auto pair_at = [&](uint32_t e, T& pe, T& po) {
      const int b = __ffs(e) - 1;
      // with minus copies (Wm = W + m NS) the update is a DADD: +1.5 % against
      // fma(+-1, col, r) (profiles/r1_walk_experiments_c0.txt)
      const bool me = StepPlan::minus_even(e, k, lane_minus);
      pe = kMinus ? step((me ? W + m * NS : W) + b * NS, 1.0) : step(W + b * NS, me ? -1.0 : 1.0);
      // shared-memory column 0: (e >> 31) is always 0; it keeps the column
      // from being hoisted out of the loop into registers (spilling the state)
      const bool mo = StepPlan::minus_odd(e + 1, k, lane_minus);
      po = C0P      ? (PK_COL0_ALIGN ? step(c0, mo ? -1.0 : 1.0) : step_c0(c0d, mo ? -1.0 : 1.0))
           : kMinus ? step((mo ? W + m * NS : W) + (e >> 31) * NS, 1.0)
                    : step(W + (e >> 31) * NS, mo ? -1.0 : 1.0);
    };
    if constexpr (kPair4) {
      // two step pairs per compensated add: d = (t0 - t1) + (t2 - t3), one
      // Neumaier step per four terms (error <= 3 u (|t0| + ... + |t3|), inside
      // the n u S gate)
      for (uint32_t e = 2; e < L; e += 4) {
        T pe, po, qe, qo;
        pair_at(e, pe, po);
        if (e + 2 < L) {
          // the second odd step reads the parameter's second copy of column 0
          // (WalkArgs::col0b): distinct uniform loads, not one copy held in
          // vector registers across the body
          const double* keep = c0d;
          c0d = c0d2;
          pair_at(e + 2, qe, qo);
          c0d = keep;
          add_quad(pe, po, qe, qo);
        } else {
          add_pair(pe, po);
        }
      }
    } else {
      // (the round-1 loop, written out: through the pair_at lambda ptxas spilled
      // the n = 44-48 complex kernels' state, 200 B against 16 B)
      for (uint32_t e = 2; e < L; e += 2) {
        const int b = __ffs(e) - 1;
        const bool me = StepPlan::minus_even(e, k, lane_minus);
        const T pe = kMinus ? step((me ? W + m * NS : W) + b * NS, 1.0)
                            : step(W + b * NS, me ? -1.0 : 1.0);
        const bool mo = StepPlan::minus_odd(e + 1, k, lane_minus);
        const T po = C0P      ? (PK_COL0_ALIGN ? step(c0, mo ? -1.0 : 1.0)
                                               : step_c0(c0d, mo ? -1.0 : 1.0))
                     : kMinus ? step((mo ? W + m * NS : W) + (e >> 31) * NS, 1.0)
                              : step(W + (e >> 31) * NS, mo ? -1.0 : 1.0);
        add_pair_blk(pe, po, ((e >> 1) & (kBlockPairs - 1)) == kBlockPairs - 1 || e + 2 >= L);
      }
    }
  }
};

// Fixed-shape butterfly over the 32 lanes (binary tree in lane order).
__device__ __forceinline__ void warp_tree(double& s, double& c) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double os = __shfl_down_sync(0xffffffffu, s, off);
    const double oc = __shfl_down_sync(0xffffffffu, c, off);
    if ((lane_id() & (2 * off - 1)) == 0) {
      const Pair p = pair_combine(Pair{s, c}, Pair{os, oc});
      s = p.s;
      c = p.c;
    }
  }
}

__device__ __forceinline__ double warp_sum_tree(double v) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double o = __shfl_down_sync(0xffffffffu, v, off);
    if ((lane_id() & (2 * off - 1)) == 0) v += o;
  }
  return v;
}

template <int N, bool CPLX, bool C0P>
__global__ void __launch_bounds__(kWalkThreads, min_ctas(N * (CPLX ? 4 : 2)))
    walk_f64_kernel(const __grid_constant__ WalkArgs args) {
  using W_ = F64Walker<N, CPLX, C0P>;
  using T = typename W_::T;
  constexpr int NS = W_::NS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const int slot_elems = ((W_::kMinus ? 2 : 1) * args.m + 1) * NS;
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  T* slot = smem + (args.per_warp_slot ? warp * slot_elems : 0);
  const size_t mat_stride = static_cast<size_t>(N) * N * (CPLX ? 2 : 1);
  const double* amat = static_cast<const double*>(args.a);

  const uint64_t units = static_cast<uint64_t>(args.B) * args.tiles;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWalkWarps + warp;
  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * kWalkWarps;

  int staged = -1;
  if (!args.per_warp_slot) {
    stage_f64<N, CPLX, W_::kMinus>(slot, amat, args.m, args.algo, threadIdx.x, blockDim.x);
    __syncthreads();
    staged = 0;
  }
  W_ w;
  w.want_abs = args.want_abs != 0;
  w.c0 = C0P ? reinterpret_cast<const T*>(args.col0) : nullptr;
  w.c0d = C0P ? args.col0 : nullptr;
#if PK_PAIR4
  w.c0d2 = C0P ? args.col0b : nullptr;
#else
  w.c0d2 = w.c0d;
#endif
  // Ryser's global sign (-1)^n: the term sign at a segment start (its Gray
  // code has even popcount).  Negation is exact and commutes with the TwoSum
  // tree, so it is applied per lane.
  const double sg0 = (args.algo == 0 && (N & 1)) ? -1.0 : 1.0;
  for (uint64_t u = gw; u < units; u += tw) {
    const int b = static_cast<int>(u / args.tiles);
    const uint64_t tl = u % args.tiles;
    if (b != staged) {  // warp-uniform; only in per-warp-slot mode
      __syncwarp();
      stage_f64<N, CPLX, W_::kMinus>(slot, amat + b * mat_stride, args.m, args.algo, lane, 32);
      __syncwarp();
      staged = b;
    }
    const uint64_t seg = ((args.tile0 + tl) << kTileBits) + lane;
    const bool active = seg < args.segs_total;
    w.walk(slot, slot + NS, args.m, args.k, active ? seg : 0);
    double s_re = 0, c_re = 0, s_im = 0, c_im = 0, ab = 0;
    if (active) {
      s_re = sg0 * w.s_re;
      c_re = sg0 * w.c_re;
      s_im = sg0 * w.s_im;
      c_im = sg0 * w.c_im;
      ab = w.abs_acc;
    }
    warp_tree(s_re, c_re);
    if constexpr (CPLX) warp_tree(s_im, c_im);
    if (args.want_abs) ab = warp_sum_tree(ab);
    if (lane == 0) {
      double* o = args.partials + (static_cast<uint64_t>(b) * args.tiles + tl) * 5;
      o[0] = s_re;
      o[1] = c_re;
      o[2] = s_im;
      o[3] = c_im;
      o[4] = ab;
    }
  }
}

// ---------------------------------------------------------------------------
// F_p walk, P primes per lane, odd p < 2^31.  The products are lazy
// Montgomery REDC trees; row sums are either kept reduced in [0, p) (add +
// min(v, v - p), one VIADDMNMX) or, when n (p - 1) < 2^31 ("lazy"), as exact
// unreduced integers (one IADD3 per row update).  One REDC costs
// IMAD.WIDE.U32 + IMAD + IMAD.HI.U32 = 5 fmaheavy issue units (measured B200
// rates: 64 IMAD, 32 IMAD.WIDE, 32 IMAD.HI lane-ops/clk/SM).
//
// Shared layout per slot (uint32): W2[2 dir][m][P][NS] (plus copy, minus copy:
// p - v reduced / -v lazy) then base[P][NS]; NS = n padded to 4 words.

template <int N, int P, bool LAZY>
__device__ void stage_modp(uint32_t* sm, const uint32_t* a, const uint32_t* primes, int m,
                           int algo, int tid, int nthreads) {
  constexpr int NS = col_stride(N, 4);
  constexpr int CS = P * NS;  // one column, all primes
  uint32_t* W = sm;
  uint32_t* base = sm + 2 * m * CS;
  const int nn = N * N;
  for (int idx = tid; idx < (m + 1) * CS; idx += nthreads) {
    const int i = idx % NS;
    const int q = (idx / NS) % P;
    const int b = idx / CS - 1;  // -1: base
    const uint32_t p = primes[q];
    const uint32_t* aq = a + q * nn;
    uint32_t v = 0;
    if (i < N) {
      if (b < 0) {
        if (algo == 1)
          for (int r = 0; r < N; ++r) {
            v += aq[r * N + i];
            v = v >= p ? v - p : v;
          }
      } else if (algo == 0) {
        v = aq[i * N + b];
      } else {
        uint32_t two = aq[(b + 1) * N + i] * 2u;  // < 2^32 since x < 2^31
        two = two >= p ? two - p : two;
        v = two == 0 ? 0u : p - two;  // -2 a[b+1][i] mod p
      }
    }
    const int off = q * NS + i;
    if (b < 0) {
      base[off] = v;
    } else {
      W[b * CS + off] = v;
      W[(m + b) * CS + off] = LAZY ? 0u - v : (v == 0 ? 0u : p - v);
    }
  }
}

// Step pairs per loop body of the F_p walks (experiment switch; 1 = the
// compiler's choice of one pair)
#ifndef PK_MODP_UNROLL
#define PK_MODP_UNROLL 1
#endif
constexpr int kModpUnroll = PK_MODP_UNROLL;

__device__ __forceinline__ uint32_t addmod_red(uint32_t r, uint32_t c, uint32_t p) {
  const uint32_t v = r + c;
  return min(v, v - p);
}

template <int N, int P, bool LAZY>
struct ModpWalker {
  static constexpr int NS = col_stride(N, 4);
  static constexpr int CS = P * NS;

  uint32_t r[P][N];
  const ModConsts* mc;              // p, -1/p, kneg (multiple of p bounding every REDC output)
  unsigned long long acc[P];        // even steps add y, odd steps kneg - y

  __device__ __forceinline__ uint32_t p(int q) const { return mc->p[q]; }

  __device__ __forceinline__ static void upd(uint32_t& r, uint32_t c, uint32_t p) {
    if constexpr (LAZY)
      r += c;
    else
      r = addmod_red(r, c, p);
  }
  // The step's row update.  PK_ALU_ADD: a third, runtime-zero operand (a
  // uniform kernel parameter) makes the add a 3-input IADD3, which only the ALU
  // pipe executes; a 2-input add may be issued as IMAD.IADD on the fmaheavy
  // pipe, the pipe the REDCs are bound by.
#ifndef PK_ALU_ADD
#define PK_ALU_ADD 0
#endif
  uint32_t zero = 0;
  __device__ __forceinline__ void upd_step(uint32_t& r, uint32_t c, uint32_t p) const {
    if constexpr (PK_ALU_ADD) {
      const uint32_t v = r + c + zero;
      r = LAZY ? v : min(v, v - p);
    } else {
      upd(r, c, p);
    }
  }

  // REDC product tree, evaluated depth-first like the fp64 tree (N - 1 REDCs,
  // scale 2^(-32 (N-1))).  Bounds: lazy rows are < 2^31 and every REDC output
  // < 2^30 + p (kneg covers it); reduced rows are < p, outputs < 2p, and a
  // merged (non-leaf) input is first brought below p so the 64-bit sum in the
  // REDC cannot overflow.
  __device__ __forceinline__ uint32_t redc2(uint32_t x, uint32_t y, bool x_leaf, int q) const {
    const uint32_t xr = (LAZY || x_leaf) ? x : min(x, x - p(q));
    return mont_lazy(xr, y, p(q), mc->mneg[q]);
  }

  __device__ __forceinline__ void tree(uint32_t* y) const {
    constexpr int LOG = 7;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      uint32_t st[LOG];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        uint32_t v = r[q][j];
        int l = 0;
#pragma unroll
        for (; l < LOG && ((j >> l) & 1); ++l) v = redc2(st[l], v, l == 0, q);
        st[l] = v;
      }
      uint32_t acc = 0;
      bool have = false;
      bool acc_leaf = false;
#pragma unroll
      for (int l = 0; l < LOG; ++l) {
        if ((N >> l) & 1) {
          if (have) {
            acc = redc2(st[l], acc, l == 0 && false, q);
            acc_leaf = false;
          } else {
            acc = st[l];
            acc_leaf = (l == 0);
            have = true;
          }
        }
      }
      (void)acc_leaf;
      y[q] = acc;
    }
  }

  // flip one column (plus or minus copy) and write the new term's products
  __device__ __forceinline__ void step(const uint32_t* __restrict__ col, uint32_t* y) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
#pragma unroll
      for (int j = 0; j < NS; j += 4) {
        const uint4 c = *reinterpret_cast<const uint4*>(col + q * NS + j);
        upd_step(r[q][j], c.x, p(q));
        if (j + 1 < N) upd_step(r[q][j + 1], c.y, p(q));
        if (j + 2 < N) upd_step(r[q][j + 2], c.z, p(q));
        if (j + 3 < N) upd_step(r[q][j + 3], c.w, p(q));
      }
    }
    tree(y);
  }

  __device__ __forceinline__ void add_pair(const uint32_t* ye, const uint32_t* yo) {
#pragma unroll
    for (int q = 0; q < P; ++q)
      acc[q] += static_cast<unsigned long long>(ye[q]) + (mc->kneg[q] - yo[q]);
  }

  __device__ __forceinline__ void walk(const uint32_t* __restrict__ W2,
                                       const uint32_t* __restrict__ base, int m, int k,
                                       uint64_t seg) {
    const uint32_t* Wm = W2 + m * CS;  // minus copies
    const uint64_t start = seg << k;
    const uint64_t g = start ^ (start >> 1);
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int j = 0; j < N; ++j) r[q][j] = base[q * NS + j];
    for (int b = k - 1; b < m; ++b) {
      if ((g >> b) & 1) {  // lane-divergent only during the start-state rebuild
        const uint32_t* col = W2 + b * CS;
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
          for (int j = 0; j < N; ++j) upd(r[q][j], col[q * NS + j], p(q));
      }
    }
#pragma unroll
    for (int q = 0; q < P; ++q) acc[q] = 0ull;
    const uint32_t L = 1u << k;
    const bool lane_minus = seg & 1;
    uint32_t ye[P], yo[P];
    tree(ye);
    step(StepPlan::minus_odd(1, k, lane_minus) ? Wm : W2, yo);
    add_pair(ye, yo);
#pragma unroll kModpUnroll
    for (uint32_t e = 2; e < L; e += 2) {
      const int b = __ffs(e) - 1;
      step((StepPlan::minus_even(e, k, lane_minus) ? Wm : W2) + b * CS, ye);
      // (e >> 31) is always 0: keeps column 0 from being hoisted into registers
      step((StepPlan::minus_odd(e + 1, k, lane_minus) ? Wm : W2) + (e >> 31) * CS, yo);
      add_pair(ye, yo);
    }
  }
};

// One prime group per launch (args.B == 1, constants in args.mc).
template <int N, int P, bool LAZY>
__global__ void __launch_bounds__(kWalkThreads, min_ctas(N * P))
    walk_modp_kernel(const __grid_constant__ WalkArgs args) {
  using W_ = ModpWalker<N, P, LAZY>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWalkWarps + warp;
  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * kWalkWarps;
  stage_modp<N, P, LAZY>(slot, static_cast<const uint32_t*>(args.a), args.mc.p, args.m, args.algo,
                         threadIdx.x, blockDim.x);
  __syncthreads();
  W_ w;
  w.mc = &args.mc;
  w.zero = static_cast<uint32_t>(args.per_warp_slot);  // always 0 for F_p launches
  unsigned long long tot[P];
#pragma unroll
  for (int q = 0; q < P; ++q) tot[q] = 0;
  for (uint64_t tl = gw; tl < args.tiles; tl += tw) {
    const uint64_t seg = ((args.tile0 + tl) << kTileBits) + lane;
    const bool active = seg < args.segs_total;
    w.walk(slot, slot + 2 * args.m * W_::CS, args.m, args.k, active ? seg : 0);
#pragma unroll
    for (int q = 0; q < P; ++q) {
      unsigned long long v = active ? w.acc[q] % args.mc.p[q] : 0ull;
      // 32 values < 2^31 -> < 2^36
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      tot[q] += v;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < P; ++q) atomicAdd(args.modp_out + q, tot[q]);
  }
}

}  // namespace pk
