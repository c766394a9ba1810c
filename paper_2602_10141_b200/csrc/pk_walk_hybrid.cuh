// F_p walk on BOTH integer pipes: the fmaheavy pipe (IMAD REDC, lazy
// Montgomery, pk_walk.cuh) and the otherwise idle FP64 pipe.
//
// The Montgomery walk is bound by the fmaheavy pipe (a REDC is 5 issue units:
// IMAD.WIDE 2 + IMAD 1 + IMAD.HI 2) while the FP64 pipe sits idle.  Here each
// lane carries PI primes on the Montgomery path and PF "fp64 primes" that use
// exact double arithmetic instead:
//   state  x  = exact unreduced row sum, 0 <= x <= n (p - 1)      (DFMA +-1: exact)
//   modmul(x, y) = h - p rint(h / p),  h = x y exact (|h| < 2^53)  (DMUL, DFMA, DADD, DFMA)
//   reduce(x)    = x - p rint(x / p)                              (DFMA, DADD, DFMA)
// with rint via the 1.5 * 2^52 shift; every product stays a signed residue with
// |y| <= p/2 + 1, so |h| <= n (p - 1)(p/2 + 1) < 2^53 whenever
// fp64_prime_ok(p, n) (p < ~2^27 / sqrt(n): 2^24.4 at n = 36).  Two row chains
// per prime hide the 32-cycle modmul link.  The lane's per-segment sums are
// exact integers in double (|acc| < 2^53).  One fp64 prime costs ~5 FP64
// instructions per row update and no fmaheavy work, so 3 Montgomery + 1 fp64
// primes cover the same CRT bits as 4 Montgomery primes at 3/4 of the
// fmaheavy time (n = 36: 3 x 25.8 + 24.4 >= 95 bits).
//
// Wide fp64 primes (WF, fp64w_prime_ok: n^2 p <= 2^50, ~2^39.7 at n = 36) use
// the FMA two-product instead of an exact h:
//   h = fl(a y), l = fma(a, y, -h)  (a y = h + l exactly)
//   modmul(a, y) = fma(-rint(h / p), p, h) + l            (6 FP64 instructions)
// The fma is exact (its true value is a small integer) and so is the final add,
// so products stay signed integers with |y| < p (bound: |y| <= p/2 + 1.5 |h| 2^-52
// and |h| <= n^2 p^2).  Chains start from the unreduced row sum, and the
// per-lane sum is reduced once per step pair (|acc| < 3p).  At ~6 + 1 FP64
// instructions per row update a wide prime carries ~40 bits against ~24.
//
// Residues of fp64 primes are plain (no Montgomery scale); Ryser's (-1)^n is
// applied on the host like for the Montgomery primes.  Residue matrices: the
// PI Montgomery primes as uint32, padded to 8 bytes, then the PF fp64 primes
// as uint64.
#pragma once

#include "pk_walk.cuh"

#ifndef PK_HYB_MINCTA
#define PK_HYB_MINCTA 2
#endif
namespace pk {

__host__ __device__ constexpr bool fp64_prime_ok(uint64_t p, int n) {
  // n (p - 1) ((p - 1) / 2 + 1) < 2^52 keeps h, its rounding shift and the
  // per-segment sums exact (conservative by a factor 2)
  return (p & 1) && p >= 3 && p < (1ull << 26) &&
         static_cast<double>(n) * static_cast<double>(p - 1) *
                 (static_cast<double>((p - 1) / 2) + 1.0) < 4503599627370496.0;
}

__host__ __device__ constexpr bool fp64w_prime_ok(uint64_t p, int n) {
  return (p & 1) && p >= 3 && p < (1ull << 50) &&
         static_cast<double>(n) * static_cast<double>(n) * static_cast<double>(p) <=
             1125899906842624.0;  // 2^50
}

template <int N, int PF, bool WF>
struct FpPart {
  static constexpr int NS = col_stride(N, 8);
  static constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52

  double x[PF][N];
  const ModConsts* mc;  // fp[q], fpinv[q]
  double acc[PF];

  __device__ __forceinline__ double reduce(double v, int q) const {
    const double qq = fma(v, mc->fpinv[q], kShift) - kShift;  // rint(v / p)
    return fma(-qq, mc->fp[q], v);
  }
  __device__ __forceinline__ double modmul(double a, double y, int q) const {
    const double h = a * y;  // exact when !WF: |h| < 2^53
    if constexpr (WF) {
      const double l = fma(a, y, -h);  // a y - h, exact
      return reduce(h, q) + l;
    } else {
      return reduce(h, q);
    }
  }

  // flip one column: x += col, col the plus or minus copy (exact integers); a
  // two-operand DADD reads fewer registers than fma(sg, col, x)
  __device__ __forceinline__ void flip(const double* __restrict__ col) {
#pragma unroll
    for (int q = 0; q < PF; ++q)
#pragma unroll
      for (int j = 0; j + 2 <= N; j += 2) {
        const double2 c = *reinterpret_cast<const double2*>(col + q * NS + j);
        x[q][j] += c.x;
        x[q][j + 1] += c.y;
      }
    if constexpr (N & 1) {
#pragma unroll
      for (int q = 0; q < PF; ++q) x[q][N - 1] += col[q * NS + N - 1];
    }
  }

  // product of the state mod p: rows dealt round-robin to kC chains (each
  // starts with a reduce), chains joined by a small tree.  A modmul link is
  // 4 dependent FP64 ops (~32 cycles), so the chains keep the critical path
  // near (N / kC + log2 kC) links.
  static constexpr int kC = N >= 16 ? 4 : (N >= 2 ? 2 : 1);

  // PK_HYB_TREE = 1 (wide primes): a depth-first binary tree over the
  // unreduced row sums, like the Montgomery tree (depth log2 N instead of
  // N / kC + log2 kC links); the two-product modmul takes leaf x leaf products
  // (|h| <= n^2 p^2, the bound fp64w_prime_ok is stated for).  It measured the
  // same as the chains (profiles/r2_hybrid_variants.txt): the walk already runs
  // at its mix ceiling (profiles/r2_hybrid_mix.txt), so the chains stay.
#ifndef PK_HYB_TREE
#define PK_HYB_TREE 0
#endif
  static constexpr bool kTree = WF && PK_HYB_TREE;

  __device__ __forceinline__ void product(double* y) const {
    if constexpr (kTree) {
      constexpr int LOG = 7;
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        double st[LOG];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double v = x[q][j];
          int l = 0;
#pragma unroll
          for (; l < LOG && ((j >> l) & 1); ++l) v = modmul(st[l], v, q);
          st[l] = v;
        }
        double acc = 0.0;
        bool have = false;
#pragma unroll
        for (int l = 0; l < LOG; ++l) {
          if ((N >> l) & 1) {
            acc = have ? modmul(st[l], acc, q) : st[l];
            have = true;
          }
        }
        y[q] = acc;
      }
      return;
    }
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      double ch[kC];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int c = i % kC;
        if (i < kC)
          ch[c] = WF ? x[q][i] : reduce(x[q][i], q);  // WF: chains start unreduced
        else
          ch[c] = modmul(x[q][i], ch[c], q);
      }
#pragma unroll
      for (int w = 1; w < kC; w *= 2)
#pragma unroll
        for (int c = 0; c + w < kC; c += 2 * w) ch[c] = modmul(ch[c], ch[c + w], q);
      y[q] = ch[0];
    }
  }
};

// Offset (in uint32 words) of the fp64 primes' uint64 residues in the group's
// residue array: the PI Montgomery matrices, padded to 8 bytes.
__host__ __device__ constexpr int hybrid_fp_offset(int pi, int n) { return (pi * n * n + 1) & ~1; }

template <int N, int PI, int PF>
__device__ void stage_hybrid(uint32_t* sm, const uint32_t* a, const uint32_t* primes,
                             const uint64_t* fprimes, int m, int algo, int tid, int nthreads) {
  // Montgomery part (lazy rows) in the layout of stage_modp; primes [0, PI)
  stage_modp<N, PI, true>(sm, a, primes, m, algo, tid, nthreads);
  // fp64 part: Wf[2 dir][m][PF][NS] (plus, minus copies) then basef[PF][NS] (doubles),
  // primes [PI, PI+PF)
  constexpr int NS4 = col_stride(N, 4);
  constexpr int NS8 = col_stride(N, 8);
  const int int_words = ((2 * m + 1) * PI * NS4 + 1) & ~1;
  double* Wf = reinterpret_cast<double*>(sm + int_words);
  double* basef = Wf + 2 * m * PF * NS8;
  const int nn = N * N;
  for (int idx = tid; idx < (m + 1) * PF * NS8; idx += nthreads) {
    const int i = idx % NS8;
    const int q = (idx / NS8) % PF;
    const int b = idx / (PF * NS8) - 1;  // -1: base
    const uint64_t p = fprimes[q];
    const uint64_t* aq =
        reinterpret_cast<const uint64_t*>(a + hybrid_fp_offset(PI, N)) + q * nn;
    uint64_t v = 0;
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
        uint64_t two = aq[(b + 1) * N + i] * 2u;
        two = two >= p ? two - p : two;
        v = two == 0 ? 0u : p - two;
      }
    }
    const double dv = static_cast<double>(v);  // exact, < 2^50
    if (b < 0) {
      basef[q * NS8 + i] = dv;
    } else {
      Wf[b * PF * NS8 + q * NS8 + i] = dv;
      Wf[(m + b) * PF * NS8 + q * NS8 + i] = -dv;
    }
  }
}

template <int N, int PI, int PF, bool WF>
struct HybridWalker {
  ModpWalker<N, PI, true> mw;
  FpPart<N, PF, WF> fw;

  __device__ __forceinline__ void walk(const uint32_t* __restrict__ W2, const uint32_t* __restrict__ base,
                                       const double* __restrict__ Wf, const double* __restrict__ basef,
                                       int m, int k, uint64_t seg) {
    constexpr int CS = ModpWalker<N, PI, true>::CS;
    constexpr int NS8 = FpPart<N, PF, WF>::NS;
    const uint32_t* Wm = W2 + m * CS;
    const double* Wfm = Wf + m * PF * NS8;  // minus copies
    const uint64_t start = seg << k;
    const uint64_t g = start ^ (start >> 1);
#pragma unroll
    for (int q = 0; q < PI; ++q)
#pragma unroll
      for (int j = 0; j < N; ++j) mw.r[q][j] = base[q * ModpWalker<N, PI, true>::NS + j];
#pragma unroll
    for (int q = 0; q < PF; ++q)
#pragma unroll
      for (int j = 0; j < N; ++j) fw.x[q][j] = basef[q * NS8 + j];
    for (int b = k - 1; b < m; ++b) {
      if ((g >> b) & 1) {
        const uint32_t* col = W2 + b * CS;
#pragma unroll
        for (int q = 0; q < PI; ++q)
#pragma unroll
          for (int j = 0; j < N; ++j) mw.r[q][j] += col[q * ModpWalker<N, PI, true>::NS + j];
        fw.flip(Wf + b * PF * NS8);
      }
    }
#pragma unroll
    for (int q = 0; q < PI; ++q) mw.acc[q] = 0ull;
#pragma unroll
    for (int q = 0; q < PF; ++q) fw.acc[q] = 0.0;
    const uint32_t L = 1u << k;
    const bool lane_minus = seg & 1;
    uint32_t ye[PI], yo[PI];
    double fe[PF], fo[PF];
    auto pair = [&]() {
      mw.add_pair(ye, yo);
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        fw.acc[q] += fe[q] - fo[q];
        if constexpr (WF) fw.acc[q] = fw.reduce(fw.acc[q], q);  // |acc| < 3p stays exact
      }
    };
    // steps 0 (no flip) and 1
    mw.tree(ye);
    fw.product(fe);
    {
      const bool mi = StepPlan::minus_odd(1, k, lane_minus);
      mw.step(mi ? Wm : W2, yo);
      fw.flip(mi ? Wfm : Wf);
      fw.product(fo);
      pair();
    }
#pragma unroll kModpUnroll
    for (uint32_t e = 2; e < L; e += 2) {
      const int b = __ffs(e) - 1;
      const bool me = StepPlan::minus_even(e, k, lane_minus);
      mw.step((me ? Wm : W2) + b * CS, ye);
      fw.flip((me ? Wfm : Wf) + b * PF * NS8);
      fw.product(fe);
      const bool mo = StepPlan::minus_odd(e + 1, k, lane_minus);
      // (e >> 31) is always 0: keeps column 0 from being hoisted into registers
      mw.step((mo ? Wm : W2) + (e >> 31) * CS, yo);
      fw.flip((mo ? Wfm : Wf) + (e >> 31) * PF * NS8);
      fw.product(fo);
      pair();
    }
  }
};

// One (Montgomery + fp64) prime group per launch (args.B == 1, constants in args.mc;
// the residue matrices of the PI Montgomery primes come first, then the fp64 ones).
template <int N, int PI, int PF, bool WF>
__global__ void __launch_bounds__(kWalkThreads, PK_HYB_MINCTA)
    walk_hybrid_kernel(const __grid_constant__ WalkArgs args) {
  constexpr int P = PI + PF;
  constexpr int NS4 = col_stride(N, 4);
  constexpr int NS8 = col_stride(N, 8);
  using HW = HybridWalker<N, PI, PF, WF>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem_raw);
  const int int_words = ((2 * args.m + 1) * PI * NS4 + 1) & ~1;
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWalkWarps + warp;
  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * kWalkWarps;
  uint64_t fpr[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) fpr[q] = static_cast<uint64_t>(args.mc.fp[q]);
  stage_hybrid<N, PI, PF>(slot, static_cast<const uint32_t*>(args.a), args.mc.p, fpr, args.m,
                          args.algo, threadIdx.x, blockDim.x);
  __syncthreads();
  HW w;
  w.mw.mc = &args.mc;
  w.fw.mc = &args.mc;
  unsigned long long tot[P];
#pragma unroll
  for (int q = 0; q < P; ++q) tot[q] = 0;
  const uint32_t* W2 = slot;
  const uint32_t* base = slot + 2 * args.m * ModpWalker<N, PI, true>::CS;
  const double* Wf = reinterpret_cast<const double*>(slot + int_words);
  const double* basef = Wf + 2 * args.m * PF * NS8;
  for (uint64_t tl = gw; tl < args.tiles; tl += tw) {
    const uint64_t seg = ((args.tile0 + tl) << kTileBits) + lane;
    const bool active = seg < args.segs_total;
    w.walk(W2, base, Wf, basef, args.m, args.k, active ? seg : 0);
#pragma unroll
    for (int q = 0; q < PI; ++q) {
      unsigned long long v = active ? w.mw.acc[q] % args.mc.p[q] : 0ull;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      tot[q] += v;
    }
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      unsigned long long v = 0;
      if (active) {
        const long long pq = static_cast<long long>(args.mc.fp[q]);
        const long long sm = static_cast<long long>(w.fw.acc[q]) % pq;  // exact integer sum
        v = static_cast<unsigned long long>(sm < 0 ? sm + pq : sm);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      tot[PI + q] += v;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < P; ++q) atomicAdd(args.modp_out + q, tot[q]);
  }
}

}  // namespace pk
