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
//             flip direction is bit (ctz(s)+1) of s, except at ctz(s) = k-1
//             where it is bit 0 of the segment index (per lane).
//   tile    = 32 consecutive segments = one warp; the warp reduces its 32
//             lanes with a fixed shuffle tree -> one partial per tile.
//   Tiles are spread over a persistent grid (grid-stride over warps); tile
//   partials are reduced by pk_reduce_tiles in a fixed, device-count
//   independent tree (fp64) or summed mod p (F_p, exact, order-free).
// The start state of a segment is rebuilt in O((m-k) n) from gray(start),
// mirroring gray.block_start_state (reference gray.py:88-114).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pk_common.cuh"

namespace pk {

constexpr int kWalkThreads = 128;  // 4 warps per CTA
constexpr int kWalkWarps = kWalkThreads / 32;

struct WalkArgs {
  const void* a;         // B matrices, row-major n x n (real f64, complex f64 interleaved, or
                         // P x n x n uint32 residues for F_p)
  int B;                 // matrices (F_p: prime groups)
  int n;                 // state length
  int m;                 // Gray bits: n (Ryser) or n-1 (Glynn)
  int algo;              // 0 Ryser, 1 Glynn
  int k;                 // segment bits (segment = 2^k indices)
  int per_warp_slot;     // 1: every warp stages its own matrix (batched mode)
  uint64_t tile0;        // first global tile index of the launch (same for every matrix)
  uint64_t tiles;        // tiles per matrix in this launch
  uint64_t segs_total;   // 2^(m-k): segments per matrix (lanes beyond are idle)
  double* partials;      // fp64: [B][tiles][5] = (s_re, c_re, s_im, c_im, abs)
  unsigned long long* modp_out;  // F_p: [B][P] raw sums (< 2^64, reduced on host)
  const uint32_t* primes;        // F_p: [B][P]
  int want_abs;          // fp64: accumulate sum |term| (parity tolerance)
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------------------
// fp64 element helpers

template <bool CPLX>
struct F64T;
template <>
struct F64T<false> {
  using T = double;
  __device__ static T zero() { return 0.0; }
  __device__ static T load(const double* a, int idx) { return a[idx]; }
};
template <>
struct F64T<true> {
  using T = double2;
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
__device__ __forceinline__ void add_if(double& r, bool on, double c) {
  const double t = r + c;
  r = on ? t : r;
}
__device__ __forceinline__ void add_if(double2& r, bool on, double2 c) {
  const double tx = r.x + c.x, ty = r.y + c.y;
  r.x = on ? tx : r.x;
  r.y = on ? ty : r.y;
}

// Neumaier step, identical in form to the reference's per-component update
// (kernels.py:56-67): t = s + v; c += (big - t) + small.
__device__ __forceinline__ void neumaier(double& s, double& c, double v) {
  const double t = s + v;
  const bool sb = fabs(s) >= fabs(v);
  const double big = sb ? s : v;
  const double small = sb ? v : s;
  c += (big - t) + small;
  s = t;
}

// Stage one matrix into shared memory in walk form: base[n] then W[m][n].
template <bool CPLX>
__device__ void stage_f64(typename F64T<CPLX>::T* sm, const double* a, int n, int m, int algo,
                          int tid, int nthreads) {
  using T = typename F64T<CPLX>::T;
  T* base = sm;
  T* W = sm + n;
  if (algo == 0) {
    for (int idx = tid; idx < n * n; idx += nthreads) {
      const int i = idx / n, b = idx % n;  // a[i][b] -> W[b][i]
      W[b * n + i] = F64T<CPLX>::load(a, idx);
    }
    for (int i = tid; i < n; i += nthreads) base[i] = F64T<CPLX>::zero();
  } else {
    for (int idx = tid; idx < (n - 1) * n; idx += nthreads) {
      const int b = idx / n, j = idx % n;  // W[b][j] = -2 a[b+1][j]
      T v = F64T<CPLX>::load(a, (b + 1) * n + j);
      if constexpr (CPLX) {
        v.x *= -2.0;
        v.y *= -2.0;
      } else {
        v *= -2.0;
      }
      W[b * n + j] = v;
    }
    for (int j = tid; j < n; j += nthreads) {
      T s = F64T<CPLX>::load(a, j);
      for (int i = 1; i < n; ++i) {
        const T v = F64T<CPLX>::load(a, i * n + j);
        if constexpr (CPLX) {
          s.x += v.x;
          s.y += v.y;
        } else {
          s += v;
        }
      }
      base[j] = s;
    }
  }
}

template <int N, bool CPLX>
struct F64Walker {
  using T = typename F64T<CPLX>::T;

  T r[N];
  double s_re, c_re, s_im, c_im, abs_acc;
  bool want_abs;

  __device__ __forceinline__ void flip(const T* __restrict__ col, double sg) {
#pragma unroll
    for (int i = 0; i < N; ++i) fma_upd(r[i], sg, col[i]);
  }

  __device__ __forceinline__ void accumulate(double pr, double pi, bool even) {
    neumaier(s_re, c_re, even ? pr : -pr);
    if constexpr (CPLX) neumaier(s_im, c_im, even ? pi : -pi);
    if (want_abs) abs_acc += fabs(pr) + (CPLX ? fabs(pi) : 0.0);
  }

  // product of the current state (no flip); even = true adds, false subtracts
  __device__ __forceinline__ void term(bool even) {
    if constexpr (CPLX) {
      double pr = r[0].x, pi = r[0].y;
#pragma unroll
      for (int i = 1; i < N; ++i) {
        const double nr = fma(pr, r[i].x, -(pi * r[i].y));
        pi = fma(pr, r[i].y, pi * r[i].x);
        pr = nr;
      }
      accumulate(pr, pi, even);
    } else {
      double p0 = r[0], p1 = N > 1 ? r[1] : 1.0;
#pragma unroll
      for (int i = 2; i < N; i += 2) {
        p0 *= r[i];
        if (i + 1 < N) p1 *= r[i + 1];
      }
      accumulate(N > 1 ? p0 * p1 : p0, 0.0, even);
    }
  }

  // flip column `col` with direction sg and accumulate the new term; the row
  // update feeds the product chain directly so column loads stay short-lived
  __device__ __forceinline__ void step(const T* __restrict__ col, double sg, bool even) {
    if constexpr (CPLX) {
      fma_upd(r[0], sg, col[0]);
      double pr = r[0].x, pi = r[0].y;
#pragma unroll
      for (int i = 1; i < N; ++i) {
        fma_upd(r[i], sg, col[i]);
        const double nr = fma(pr, r[i].x, -(pi * r[i].y));
        pi = fma(pr, r[i].y, pi * r[i].x);
        pr = nr;
      }
      accumulate(pr, pi, even);
    } else {
      // two interleaved chains hide DMUL latency
      fma_upd(r[0], sg, col[0]);
      double p0 = r[0], p1 = 1.0;
#pragma unroll
      for (int i = 1; i < N; ++i) {
        fma_upd(r[i], sg, col[i]);
        if (i & 1)
          p1 = (i == 1) ? r[i] : p1 * r[i];
        else
          p0 *= r[i];
      }
      accumulate(N > 1 ? p0 * p1 : p0, 0.0, even);
    }
  }

  // Walk segment `seg` (2^k indices starting at seg << k).
  __device__ __forceinline__ void walk(const T* __restrict__ base, const T* __restrict__ W,
                                       int m, int k, uint64_t seg) {
    const uint64_t start = seg << k;
    const uint64_t g = start ^ (start >> 1);
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = base[i];
    for (int j = (k > 0 ? k - 1 : 0); j < m; ++j) {
      const bool on = (g >> j) & 1;
      const T* col = W + j * N;
#pragma unroll
      for (int i = 0; i < N; ++i) add_if(r[i], on, col[i]);
    }
    s_re = c_re = s_im = c_im = abs_acc = 0.0;
    term(true);
    const uint32_t L = 1u << k;
    const double lane_sg = (seg & 1) ? -1.0 : 1.0;  // direction at ctz = k-1
    const double sg_odd0 = (k == 1) ? lane_sg : 1.0;
    for (uint32_t s = 1; s + 1 < L; s += 2) {
      // odd step s: column 0, direction = bit 1 of s (k >= 2 here).  The
      // (s >> 31) term (always 0) keeps the compiler from hoisting column 0
      // out of the loop into registers, which would spill the state.
      step(W + (s >> 31) * N, ((s >> 1) & 1) ? -1.0 : 1.0, false);
      // even step s+1: column b = ctz(s+1) >= 1
      const uint32_t e = s + 1;
      const int b = __ffs(e) - 1;
      const double sg = (b == k - 1) ? lane_sg : (((e >> (b + 1)) & 1) ? -1.0 : 1.0);
      step(W + b * N, sg, true);
    }
    // last odd step s = L-1 (bit 1 set when k >= 2)
    step(W, (k == 1) ? sg_odd0 : -1.0, false);
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

template <int N, bool CPLX>
__global__ void __launch_bounds__(kWalkThreads, 2) walk_f64_kernel(WalkArgs args) {
  using T = typename F64T<CPLX>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const int slot_elems = N + N * args.m;  // base + W
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
    stage_f64<CPLX>(slot, amat, N, args.m, args.algo, threadIdx.x, blockDim.x);
    __syncthreads();
    staged = 0;
  }
  F64Walker<N, CPLX> w;
  w.want_abs = args.want_abs != 0;
  for (uint64_t u = gw; u < units; u += tw) {
    const int b = static_cast<int>(u / args.tiles);
    const uint64_t tl = u % args.tiles;
    if (b != staged) {  // warp-uniform; only in per-warp-slot mode
      __syncwarp();
      stage_f64<CPLX>(slot, amat + b * mat_stride, N, args.m, args.algo, lane, 32);
      __syncwarp();
      staged = b;
    }
    const uint64_t seg = ((args.tile0 + tl) << 5) + lane;
    const bool active = seg < args.segs_total;
    double s_re = 0, c_re = 0, s_im = 0, c_im = 0, ab = 0;
    w.walk(slot, slot + N, args.m, args.k, active ? seg : 0);
    if (active) {
      // Ryser's global sign (-1)^n (the term sign at a segment start, whose
      // Gray code has even popcount); negation is exact and commutes with
      // the TwoSum tree, so it is applied per lane.
      const double sg0 = (args.algo == 0 && (N & 1)) ? -1.0 : 1.0;
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
// F_p walk, P primes per lane, p < 2^31 odd.  State residues are kept reduced
// in [0, p) (add, then min(v, v-p)); the product chain is lazy Montgomery
// (values in [0, 2p)), so one row update costs IADD3 + IMNMX (ALU pipe) and
// one multiply costs 3 IMAD-class instructions (FMA pipe).
//
// Shared layout per slot (uint32): W2[2][m][P][NP] (plus-column, p-minus
// column) then base[P][NP]; NP = N rounded up to 4 for 16-byte broadcast loads.

template <int N>
struct NPad {
  static constexpr int v = (N + 3) & ~3;
};

template <int N, int P, bool LAZY>
__device__ void stage_modp(uint32_t* sm, const uint32_t* a, const uint32_t* primes, int m,
                           int algo, int tid, int nthreads) {
  constexpr int NP = NPad<N>::v;
  uint32_t* W = sm;                     // [2][m][P][NP]
  uint32_t* base = sm + 2 * m * P * NP;  // [P][NP]
  const int nn = N * N;
  for (int idx = tid; idx < m * P * NP; idx += nthreads) {
    const int i = idx % NP;
    const int q = (idx / NP) % P;
    const int b = idx / (NP * P);
    const uint32_t p = primes[q];
    uint32_t v = 0;
    if (i < N) {
      if (algo == 0) {
        v = a[q * nn + i * N + b];  // column b, row i
      } else {
        const uint32_t x = a[q * nn + (b + 1) * N + i];
        uint32_t two = x + x;  // < 2^32 since x < 2^31
        two = two >= p ? two - p : two;
        v = two == 0 ? 0 : p - two;  // -2 a[b+1][i] mod p
      }
    }
    W[(0 * m + b) * P * NP + q * NP + i] = v;
    // minus copy: p - v (reduced state) or the two's complement -v (lazy state,
    // exact integer sums: r - v never wraps because v was added before)
    W[(1 * m + b) * P * NP + q * NP + i] = (i < N) ? (LAZY ? 0u - v : (v == 0 ? 0 : p - v)) : 0;
  }
  for (int idx = tid; idx < P * NP; idx += nthreads) {
    const int i = idx % NP, q = idx / NP;
    const uint32_t p = primes[q];
    uint32_t s = 0;
    if (algo == 1 && i < N) {
      for (int r = 0; r < N; ++r) {
        s += a[q * nn + r * N + i];
        s = s >= p ? s - p : s;
      }
    }
    base[q * NP + i] = s;
  }
}

__device__ __forceinline__ uint32_t addmod_red(uint32_t r, uint32_t c, uint32_t p) {
  const uint32_t v = r + c;
  return min(v, v - p);
}

template <int N, int P, bool LAZY>
struct ModpWalker {
  static constexpr int NP = NPad<N>::v;
  uint32_t r[P][N];
  uint32_t p[P], mneg[P], kneg[P];  // kneg: multiple of p bounding every product y
  // even steps add y, odd steps add kneg - y (y <= kneg), so one 64-bit
  // accumulator carries (even - odd) mod p without a negation per term
  unsigned long long acc[P];

  // lazy: exact integer row sums (n p < 2^31), one IADD3; reduced: [0, p)
  __device__ __forceinline__ static void upd(uint32_t& r, uint32_t c, uint32_t p) {
    if constexpr (LAZY)
      r += c;
    else
      r = addmod_red(r, c, p);
  }

  __device__ __forceinline__ void flip(const uint32_t* __restrict__ col) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const uint4* c4 = reinterpret_cast<const uint4*>(col + q * NP);
#pragma unroll
      for (int i4 = 0; i4 < NP / 4; ++i4) {
        const uint4 c = c4[i4];
        if (4 * i4 + 0 < N) upd(r[q][4 * i4 + 0], c.x, p[q]);
        if (4 * i4 + 1 < N) upd(r[q][4 * i4 + 1], c.y, p[q]);
        if (4 * i4 + 2 < N) upd(r[q][4 * i4 + 2], c.z, p[q]);
        if (4 * i4 + 3 < N) upd(r[q][4 * i4 + 3], c.w, p[q]);
      }
    }
  }

  __device__ __forceinline__ void term(bool even) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
      uint32_t y;
      if constexpr (N == 1) {
        y = r[q][0];
      } else {
        y = mont_lazy(r[q][0], r[q][1], p[q], mneg[q]);
#pragma unroll
        for (int i = 2; i < N; ++i) y = mont_lazy(r[q][i], y, p[q], mneg[q]);
      }
      acc[q] += even ? y : (kneg[q] - y);
    }
  }

  // W2 = [2][m][P][NP]; direction d selects the plus (0) or minus (1) copy.
  __device__ __forceinline__ void walk(const uint32_t* __restrict__ W2,
                                       const uint32_t* __restrict__ base, int m, int k,
                                       uint64_t seg) {
    const int colstride = P * NP;
    const uint32_t* Wm = W2 + m * colstride;  // minus copies
    const uint64_t start = seg << k;
    const uint64_t g = start ^ (start >> 1);
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int i = 0; i < N; ++i) r[q][i] = base[q * NP + i];
    for (int j = (k > 0 ? k - 1 : 0); j < m; ++j) {
      if ((g >> j) & 1) flip(W2 + j * colstride);  // lane-divergent only during init
    }
#pragma unroll
    for (int q = 0; q < P; ++q) acc[q] = 0ull;
    term(true);
    const uint32_t L = 1u << k;
    const bool lane_minus = seg & 1;
    for (uint32_t s = 1; s + 1 < L; s += 2) {
      flip((((s >> 1) & 1) ? Wm : W2) + (s >> 31) * colstride);  // see fp64 walker
      term(false);
      const uint32_t e = s + 1;
      const int b = __ffs(e) - 1;
      const bool minus = (b == k - 1) ? lane_minus : ((e >> (b + 1)) & 1);
      flip((minus ? Wm : W2) + b * colstride);
      term(true);
    }
    flip((k == 1) ? (lane_minus ? Wm : W2) : Wm);
    term(false);
  }
};

template <int N, int P, bool LAZY>
__global__ void __launch_bounds__(kWalkThreads) walk_modp_kernel(WalkArgs args) {
  constexpr int NP = NPad<N>::v;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* smem = reinterpret_cast<uint32_t*>(smem_raw);
  const int slot_words = (2 * args.m + 1) * P * NP;
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  uint32_t* slot = smem + (args.per_warp_slot ? warp * slot_words : 0);
  const uint32_t* amat = static_cast<const uint32_t*>(args.a);
  const size_t mat_stride = static_cast<size_t>(P) * N * N;

  const uint64_t units = static_cast<uint64_t>(args.B) * args.tiles;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWalkWarps + warp;
  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * kWalkWarps;

  int staged = -1;
  if (!args.per_warp_slot) {
    stage_modp<N, P, LAZY>(slot, amat, args.primes, args.m, args.algo, threadIdx.x, blockDim.x);
    __syncthreads();
    staged = 0;
  }
  ModpWalker<N, P, LAZY> w;
  unsigned long long tot[P];
#pragma unroll
  for (int q = 0; q < P; ++q) tot[q] = 0;
  int cur_b = -1;
  for (uint64_t u = gw; u < units; u += tw) {
    const int b = static_cast<int>(u / args.tiles);
    const uint64_t tl = u % args.tiles;
    if (b != cur_b) {
      if (cur_b >= 0 && lane == 0) {
#pragma unroll
        for (int q = 0; q < P; ++q) atomicAdd(args.modp_out + cur_b * P + q, tot[q]);
      }
#pragma unroll
      for (int q = 0; q < P; ++q) tot[q] = 0;
      cur_b = b;
#pragma unroll
      for (int q = 0; q < P; ++q) {
        w.p[q] = args.primes[b * P + q];
        w.mneg[q] = mont_neg_inv32(w.p[q]);
        // products stay below 2p (reduced state) or below (n/2 + 2) p (lazy
        // state, n p <= 2^31: the first REDC sees two unreduced sums)
        w.kneg[q] = LAZY ? w.p[q] * static_cast<uint32_t>(N / 2 + 2) : 2u * w.p[q];
      }
    }
    if (b != staged) {
      __syncwarp();
      stage_modp<N, P, LAZY>(slot, amat + b * mat_stride, args.primes + b * P, args.m, args.algo, lane,
                       32);
      __syncwarp();
      staged = b;
    }
    const uint64_t seg = ((args.tile0 + tl) << 5) + lane;
    const bool active = seg < args.segs_total;
    w.walk(slot, slot + 2 * args.m * P * NP, args.m, args.k, active ? seg : 0);
#pragma unroll
    for (int q = 0; q < P; ++q) {
      unsigned long long v = w.acc[q] % w.p[q];
      v = active ? v : 0ull;
      // lane sum: 32 values < 2^32 -> < 2^37
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      tot[q] += v;
    }
  }
  if (cur_b >= 0 && lane == 0) {
#pragma unroll
    for (int q = 0; q < P; ++q) atomicAdd(args.modp_out + cur_b * P + q, tot[q]);
  }
}

}  // namespace pk
