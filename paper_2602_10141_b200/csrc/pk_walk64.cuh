// F_p walk for wide odd moduli 2^31 <= p < 2^62: the reference's default CRT
// basis (59-bit primes, modular.py:25, 100-108) and any PrimeField modulus that
// does not fit the 32-bit Montgomery kernels (domains.py:126-130).
//
// Same Gray skeleton as walk_modp_kernel (pk_walk.cuh): aligned 2^k-step
// segments per lane, warp-uniform flip column from shared memory, plus / minus
// column copies selected by the step direction, depth-first product tree.
// Arithmetic is Montgomery with R = 2^64 and the positive inverse
// p' = p^-1 mod 2^64:
//     T = x y = hi 2^64 + lo,  m = lo p' mod 2^64  =>  m p = lo (mod 2^64)
//     REDC(T) = (T - m p) / 2^64 = hi - umulhi(m, p)      in (-p, p)
// so no low-word add or carry is needed; adding p gives (0, 2p).  Inputs below
// 2p keep T < 4p^2 < p 2^64 (p < 2^62), so REDC outputs can feed the next
// REDC unreduced.  One REDC = two 64-bit low products and two 64-bit high
// products on the fmaheavy pipe (~20 issue units, against 5 for Montgomery-32).
//
// Row sums stay reduced in [0, p) (64-bit add + conditional subtract on the
// ALU pipe).  Each lane accumulates its segment's signed terms exactly in 128
// bits and folds them once per segment with one more REDC; warps combine mod p
// and add into a 128-bit (lo, hi) counter per prime with a carry-propagating
// atomic pair.  The host multiplies by 2^(64 n) (the tree's 2^(-64 (n-1)) and
// the fold's 2^-64) and applies Ryser's (-1)^n.
#pragma once

#include "pk_walk.cuh"

namespace pk {

// Steps per loop body: two (the round-2 REDC made a step ~1,180 instructions;
// the two-step body measured +4-5 % at n = 35 / 36 with no instruction-cache
// stalls, where round 1's ~1,500-instruction steps thrashed it;
// profiles/r2_wide_variants.txt)
#ifndef PK_WIDE_UNROLL
#define PK_WIDE_UNROLL 2
#endif
constexpr int kWideUnroll = PK_WIDE_UNROLL;
#ifndef PK_REDC64_WIDE_E
#define PK_REDC64_WIDE_E 0  // experiment: hi(m0 p0) from a wide multiply
#endif

__device__ __forceinline__ uint64_t wmul32(uint32_t a, uint32_t b) {
  return static_cast<uint64_t>(a) * b;  // IMAD.WIDE.U32
}
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return static_cast<uint32_t>(v); }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return static_cast<uint32_t>(v >> 32); }

// REDC(x y) = x y 2^-64 mod p in (0, 2p), for x y < p 2^64 (x, y < 2^63).
// Schoolbook over 32-bit limbs, arranged so that no addend needs a
// zero-extended register pair (a 64-bit addend of IMAD.WIDE.U32 is a register
// pair; zero-extending a 32-bit word into one costs two extra instructions):
//   x y:  lo = x0 y0, mid = x0 y1 + x1 y0 (< 2^64 for x, y < 2^63: the second
//         multiply takes the first as its addend), hi = x1 y1; the 64-bit
//         halves follow with one add.cc / addc / addc carry chain;
//   m  = lo64(x y) p' mod 2^64: one wide and two plain IMADs;
//   hi64(m p): m1 p0 + (m0 p1 + hi(m0 p0)) is 65 bits: add.cc / addc / addc,
//         then added to m1 p1 (its low 64 bits equal lo64(x y): no borrow).
// 8 IMAD.WIDE.U32 + 1 IMAD.HI.U32 + 2 IMAD (40 fmaheavy SMSP cycles per warp)
// and 8 carry-chain ALU instructions.
// Word-serial Montgomery (CIOS) with two 32-bit rounds and the same R = 2^64:
// m_i = t_i (-p^-1) mod 2^32, T += m_i p, T >>= 32.  8 IMAD.WIDE + 2 IMAD (36
// fmaheavy cycles against redc64_lazy's 40) and ~15 carry adds on the ALU pipe,
// which has room.  Output in [0, 2p) for x y < p 2^64 (T + m p < 2^127 for
// p < 2^62).  Measured +4-6 % over redc64_lazy's form at n = 32-36
// (profiles/r2_wide_variants.txt): the default.
#ifndef PK_REDC64_CIOS
#define PK_REDC64_CIOS 1
#endif
__device__ __forceinline__ uint64_t redc64_cios(uint64_t x, uint64_t y, uint64_t p,
                                                uint64_t pinv) {
  uint64_t r;
  asm("{\n\t"
      ".reg .u32 x0, x1, y0, y1, p0, p1, q0, q1, t0, t1, t2, t3, m0, m1, z;\n\t"
      ".reg .u32 a0, a1, b0, b1, c0, c1, d0, d1, h0, h1, s0, s1;\n\t"
      ".reg .u64 lo, mid, hi, a, b, c, d;\n\t"
      "mov.b64 {x0, x1}, %1;\n\t"
      "mov.b64 {y0, y1}, %2;\n\t"
      "mov.b64 {p0, p1}, %3;\n\t"
      "mov.b64 {q0, q1}, %4;\n\t"
      "neg.s32 q0, q0;\n\t"  // -p^-1 mod 2^32 from the positive inverse
      // T = x y = (t3 t2 t1 t0)
      "mul.wide.u32 lo, x0, y0;\n\t"
      "mul.wide.u32 mid, x0, y1;\n\t"
      "mad.wide.u32 mid, x1, y0, mid;\n\t"
      "mul.wide.u32 hi, x1, y1;\n\t"
      "mov.b64 {t0, t1}, lo;\n\t"
      "mov.b64 {s0, s1}, mid;\n\t"
      "mov.b64 {h0, h1}, hi;\n\t"
      "add.cc.u32 t1, t1, s0;\n\t"
      "addc.cc.u32 t2, h0, s1;\n\t"
      "addc.u32 t3, h1, 0;\n\t"
      // round 1: T += m0 p, drop t0
      "mul.lo.u32 m0, t0, q0;\n\t"
      "mul.wide.u32 a, m0, p0;\n\t"
      "mul.wide.u32 b, m0, p1;\n\t"
      "mov.b64 {a0, a1}, a;\n\t"
      "mov.b64 {b0, b1}, b;\n\t"
      "add.cc.u32 z, t0, a0;\n\t"  // 0 mod 2^32: only the carry
      "addc.cc.u32 t1, t1, a1;\n\t"
      "addc.cc.u32 t2, t2, 0;\n\t"
      "addc.u32 t3, t3, 0;\n\t"
      "add.cc.u32 t1, t1, b0;\n\t"
      "addc.cc.u32 t2, t2, b1;\n\t"
      "addc.u32 t3, t3, 0;\n\t"
      // round 2: T += m1 p 2^32, drop t1
      "mul.lo.u32 m1, t1, q0;\n\t"
      "mul.wide.u32 c, m1, p0;\n\t"
      "mul.wide.u32 d, m1, p1;\n\t"
      "mov.b64 {c0, c1}, c;\n\t"
      "mov.b64 {d0, d1}, d;\n\t"
      "add.cc.u32 z, t1, c0;\n\t"
      "addc.cc.u32 t2, t2, c1;\n\t"
      "addc.u32 t3, t3, 0;\n\t"
      "add.cc.u32 t2, t2, d0;\n\t"
      "addc.u32 t3, t3, d1;\n\t"
      "mov.b64 %0, {t2, t3};\n\t"
      "}"
      : "=l"(r)
      : "l"(x), "l"(y), "l"(p), "l"(pinv));
  return r;
}

// Lazy-walk REDC (p < 2^60, x, y < 4p < 2^62), word-serial like redc64_cios but
// with the 64-bit column sums kept in IMAD.WIDE addends, which the bounds allow:
//   mid = x0 y1 + x1 y0 < 2^63, A = mid + m0 p1 < 2^63.2 (p1 < 2^28), and
//   digit 0 of T + m0 p is lo_lo + lo32(m0 p0) = 0 or 2^32: its carry is
//   (lo_lo != 0), so only hi32(m0 p0) is formed (IMAD.HI, same cost as a wide).
//   U = (T + m0 p) / 2^32 = S + hi 2^32, S = A + lo_hi + hi32(m0 p0) + c0 < 2^64;
//   result = (U + m1 p) / 2^32 = (m1 p1 + hi) + hi32(S) + hi32(m1 p0) + c1.
// Same fmaheavy cost as CIOS (6 IMAD.WIDE + 2 IMAD.HI + 2 IMAD), 10 carry adds
// instead of 15.  Output in [0, 2p) for x y < p 2^64.  Measured +5-6 % over
// CIOS at n = 35 / 36 (0.69 -> 0.73e12 prime-row-updates/s); form 2 folds the
// 32-bit addend and digit 0's carry into the high product (madc.hi.cc: no
// zeroed addend register per IMAD.HI), another +2 % (0.75e12,
// profiles/r2_redc_ps.txt): the default for the lazy walk.  CIOS stays for
// 2^60 <= p < 2^62, where the column sums would overflow.
#ifndef PK_REDC64_PS
#define PK_REDC64_PS 2
#endif
__device__ __forceinline__ uint64_t redc64_ps(uint64_t x, uint64_t y, uint64_t p,
                                              uint64_t pinv) {
  uint64_t r;
  asm("{\n\t"
      ".reg .u32 x0, x1, y0, y1, p0, p1, q0, q1, m0, m1, l0, l1, h0, h1, z, s0, s1, r0, r1;\n\t"
      ".reg .u64 lo, A, hi, R;\n\t"
      "mov.b64 {x0, x1}, %1;\n\t"
      "mov.b64 {y0, y1}, %2;\n\t"
      "mov.b64 {p0, p1}, %3;\n\t"
      "mov.b64 {q0, q1}, %4;\n\t"
      "neg.s32 q0, q0;\n\t"  // -p^-1 mod 2^32 from the positive inverse
      "mul.wide.u32 lo, x0, y0;\n\t"
      "mul.wide.u32 A, x0, y1;\n\t"
      "mad.wide.u32 A, x1, y0, A;\n\t"
      "mul.wide.u32 hi, x1, y1;\n\t"
      "mov.b64 {l0, l1}, lo;\n\t"
      "mul.lo.u32 m0, l0, q0;\n\t"
      "mad.wide.u32 A, m0, p1, A;\n\t"
      "mov.b64 {s0, s1}, A;\n\t"
#if PK_REDC64_PS == 2
      // h0 = hi(m0 p0) + l1 + c0 in one extended-precision multiply-add; its
      // carry has weight 2^32, i.e. goes straight into s1
      "add.cc.u32 z, l0, 0xffffffff;\n\t"  // carry = (l0 != 0)
      "madc.hi.cc.u32 h0, m0, p0, l1;\n\t"
      "addc.u32 s1, s1, 0;\n\t"
      "add.cc.u32 s0, s0, h0;\n\t"
      "addc.u32 s1, s1, 0;\n\t"
      "mul.lo.u32 m1, s0, q0;\n\t"
      "mad.wide.u32 R, m1, p1, hi;\n\t"
      "mov.b64 {r0, r1}, R;\n\t"
      "add.cc.u32 z, s0, 0xffffffff;\n\t"  // carry = (s0 != 0)
      "madc.hi.cc.u32 h1, m1, p0, s1;\n\t"
      "addc.u32 r1, r1, 0;\n\t"
      "add.cc.u32 r0, r0, h1;\n\t"
      "addc.u32 r1, r1, 0;\n\t"
#else
      "mul.hi.u32 h0, m0, p0;\n\t"
      "add.cc.u32 z, l0, 0xffffffff;\n\t"  // carry = (l0 != 0)
      "addc.cc.u32 s0, s0, l1;\n\t"
      "addc.u32 s1, s1, 0;\n\t"
      "add.cc.u32 s0, s0, h0;\n\t"
      "addc.u32 s1, s1, 0;\n\t"
      "mul.lo.u32 m1, s0, q0;\n\t"
      "mad.wide.u32 R, m1, p1, hi;\n\t"
      "mul.hi.u32 h1, m1, p0;\n\t"
      "mov.b64 {r0, r1}, R;\n\t"
      "add.cc.u32 z, s0, 0xffffffff;\n\t"  // carry = (s0 != 0)
      "addc.cc.u32 r0, r0, s1;\n\t"
      "addc.u32 r1, r1, 0;\n\t"
      "add.cc.u32 r0, r0, h1;\n\t"
      "addc.u32 r1, r1, 0;\n\t"
#endif
      "mov.b64 %0, {r0, r1};\n\t"
      "}"
      : "=l"(r)
      : "l"(x), "l"(y), "l"(p), "l"(pinv));
  return r;
}

__device__ __forceinline__ uint64_t redc64_lazy(uint64_t x, uint64_t y, uint64_t p,
                                                uint64_t pinv) {
  if constexpr (PK_REDC64_CIOS) return redc64_cios(x, y, p, pinv);
  // one PTX block: left to the front end, the 64-bit adds of zero-extended
  // words survived as VIADD-with-zero register copies (~5 per REDC)
  uint64_t r;
  asm("{\n\t"
      ".reg .u32 x0, x1, y0, y1, p0, p1, q0, q1, l0, l1, d0, d1, m0, m1, t, e;\n\t"
      ".reg .u32 a0, a1, b0, b1, w0, w1, s0, s1, c, h0, h1, r0, r1;\n\t"
      ".reg .u64 lo, mid, hi, u0, a, b, w;\n\t"
      "mov.b64 {x0, x1}, %1;\n\t"
      "mov.b64 {y0, y1}, %2;\n\t"
      "mov.b64 {p0, p1}, %3;\n\t"
      "mov.b64 {q0, q1}, %4;\n\t"
      // x y = lo + mid 2^32 + hi 2^64
      "mul.wide.u32 lo, x0, y0;\n\t"
      "mul.wide.u32 mid, x0, y1;\n\t"
      "mad.wide.u32 mid, x1, y0, mid;\n\t"
      "mul.wide.u32 hi, x1, y1;\n\t"
      "mov.b64 {l0, t}, lo;\n\t"
      "mov.b64 {s0, s1}, mid;\n\t"
      "mov.b64 {w0, w1}, hi;\n\t"
      "add.cc.u32 l1, t, s0;\n\t"
      "addc.cc.u32 d0, w0, s1;\n\t"
      "addc.u32 d1, w1, 0;\n\t"
      // m = (l1 l0) p' mod 2^64
      "mul.wide.u32 u0, l0, q0;\n\t"
      "mov.b64 {m0, t}, u0;\n\t"
      "mad.lo.u32 t, l0, q1, t;\n\t"
      "mad.lo.u32 m1, l1, q0, t;\n\t"
      // high 64 bits of m p = m1 p1 + (m1 p0 + m0 p1 + hi(m0 p0)) >> 32
      "mul.wide.u32 a, m1, p0;\n\t"
      "mul.wide.u32 b, m0, p1;\n\t"
#if PK_REDC64_WIDE_E
      "mul.wide.u32 w, m0, p0;\n\t"  // (w reused below) only its high word matters
      "mov.b64 {s1, e}, w;\n\t"
#else
      "mul.hi.u32 e, m0, p0;\n\t"
#endif
      "mul.wide.u32 w, m1, p1;\n\t"
      "mov.b64 {a0, a1}, a;\n\t"
      "mov.b64 {b0, b1}, b;\n\t"
      "mov.b64 {w0, w1}, w;\n\t"
      "add.cc.u32 s0, a0, b0;\n\t"
      "addc.cc.u32 s1, a1, b1;\n\t"
      "addc.u32 c, 0, 0;\n\t"
      "add.cc.u32 s0, s0, e;\n\t"
      "addc.cc.u32 s1, s1, 0;\n\t"
      "addc.u32 c, c, 0;\n\t"
      "add.cc.u32 h0, w0, s1;\n\t"
      "addc.u32 h1, w1, c;\n\t"
      // d - h + p in (0, 2p): lo(m p) = lo(x y), so no borrow from below
      "sub.cc.u32 r0, d0, h0;\n\t"
      "subc.u32 r1, d1, h1;\n\t"
      "add.cc.u32 r0, r0, p0;\n\t"
      "addc.u32 r1, r1, p1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t"
      "}"
      : "=l"(r)
      : "l"(x), "l"(y), "l"(p), "l"(pinv));
  return r;
}

__device__ __forceinline__ uint64_t min_u64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// (hi 2^64 + lo) 2^-64 mod p in [0, p), for hi < p
__device__ __forceinline__ uint64_t fold128(uint64_t lo, uint64_t hi, uint64_t p, uint64_t pinv) {
  const uint64_t t = __umul64hi(lo * pinv, p);
  return hi >= t ? hi - t : hi - t + p;
}

// Shared layout per slot (uint64): W2[2 dir][m][P][NS] then base[P][NS], NS = n
// padded to 2 words (16-byte column loads).
template <int N, int P>
__device__ void stage_modp64(uint64_t* sm, const uint64_t* a, const uint64_t* primes, int m,
                             int algo, int tid, int nthreads) {
  constexpr int NS = col_stride(N, 8);
  constexpr int CS = P * NS;
  uint64_t* W = sm;
  uint64_t* base = sm + 2 * m * CS;
  const int nn = N * N;
  for (int idx = tid; idx < (m + 1) * CS; idx += nthreads) {
    const int i = idx % NS;
    const int q = (idx / NS) % P;
    const int b = idx / CS - 1;  // -1: base
    const uint64_t p = primes[q];
    const uint64_t* aq = a + q * nn;
    uint64_t v = 0;
    if (i < N) {
      if (b < 0) {
        if (algo == 1)
          for (int r = 0; r < N; ++r) {
            v += aq[r * N + i];  // < 2p < 2^63
            v = v >= p ? v - p : v;
          }
      } else if (algo == 0) {
        v = aq[i * N + b];
      } else {
        uint64_t two = aq[(b + 1) * N + i] * 2ull;
        two = two >= p ? two - p : two;
        v = two == 0 ? 0ull : p - two;  // -2 a[b+1][i] mod p
      }
    }
    const int off = q * NS + i;
    if (b < 0) {
      base[off] = v;
    } else {
      W[b * CS + off] = v;
      W[(m + b) * CS + off] = v == 0 ? 0ull : p - v;
    }
  }
}

// LAZY (p < 2^60): rows are reduced only on every second step.  Invariant:
// rows < 2p after a reduction; a flip adds < p + 1 (plus copy v < p, minus
// copy p - v <= p), so the tree sees rows < 3p (odd steps) or < 4p (even
// steps, reduced after their tree by one conditional subtraction of 2p), and
// 16 p^2 < p 2^64 keeps every REDC output in (0, 2p).  A flip is then a plain
// 64-bit add (2 ALU) plus half a reduction (6 ALU / 2), against 8 ALU for the
// reduced form min(v, v - p).
template <int N, int P, bool LAZY>
struct Modp64Walker {
  static constexpr int NS = col_stride(N, 8);
  static constexpr int CS = P * NS;

  uint64_t r[P][N];
  uint64_t zero = 0;  // a runtime zero (PK_ALU_ADD)
  const ModConsts* mc;
  uint64_t acc_lo[P], acc_hi[P];  // exact 128-bit sum of the segment's terms

  __device__ __forceinline__ uint64_t p(int q) const { return mc->p64[q]; }
  __device__ __forceinline__ uint64_t redc(uint64_t x, uint64_t y, int q) const {
    if constexpr (LAZY && PK_REDC64_PS) return redc64_ps(x, y, p(q), mc->pinv64[q]);
    return redc64_lazy(x, y, p(q), mc->pinv64[q]);
  }

  __device__ __forceinline__ static void upd(uint64_t& r, uint64_t c, uint64_t p) {
    const uint64_t v = r + c;  // < 2p < 2^63
    r = min_u64(v, v - p);
  }

  __device__ __forceinline__ void tree(uint64_t* y) const {
    constexpr int LOG = 7;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      uint64_t st[LOG];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        uint64_t v = r[q][j];
        int l = 0;
#pragma unroll
        for (; l < LOG && ((j >> l) & 1); ++l) v = redc(st[l], v, q);
        st[l] = v;
      }
      uint64_t acc = 0;
      bool have = false;
#pragma unroll
      for (int l = 0; l < LOG; ++l) {
        if ((N >> l) & 1) {
          if (have) {
            acc = redc(st[l], acc, q);
          } else {
            acc = st[l];
            have = true;
          }
        }
      }
      y[q] = acc;  // < 2p
    }
  }

  __device__ __forceinline__ void step(const uint64_t* __restrict__ col, uint64_t* y) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
#pragma unroll
      for (int j = 0; j < NS; j += 2) {
        const ulonglong2 c = *reinterpret_cast<const ulonglong2*>(col + q * NS + j);
        upd(r[q][j], c.x, p(q));
        if (j + 1 < N) upd(r[q][j + 1], c.y, p(q));
      }
    }
    tree(y);
  }

  // even steps add y, odd steps add 2p - y (both < 2p + 1 <= 2^63)
  __device__ __forceinline__ void add_pair(const uint64_t* ye, const uint64_t* yo) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const uint64_t v = ye[q] + (2 * p(q) - yo[q]);  // < 4p < 2^64
      const uint64_t lo = acc_lo[q] + v;
      acc_hi[q] += lo < v ? 1ull : 0ull;
      acc_lo[q] = lo;
    }
  }

  __device__ __forceinline__ void walk(const uint64_t* __restrict__ W2,
                                       const uint64_t* __restrict__ base, int m, int k,
                                       uint64_t seg) {
    const uint64_t* Wm = W2 + m * CS;
    const uint64_t start = seg << k;
    const uint64_t g = start ^ (start >> 1);
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int j = 0; j < N; ++j) r[q][j] = base[q * NS + j];
    for (int b = k - 1; b < m; ++b) {
      if ((g >> b) & 1) {
        const uint64_t* col = W2 + b * CS;
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
          for (int j = 0; j < N; ++j) upd(r[q][j], col[q * NS + j], p(q));
      }
    }
#pragma unroll
    for (int q = 0; q < P; ++q) acc_lo[q] = acc_hi[q] = 0ull;
    const uint32_t L = 1u << k;
    const bool lane_minus = seg & 1;
    // Round 1 kept one step (one product tree) per loop body: its REDC-64 tree
    // was ~1,500 instructions and a two-step body overflowed the instruction
    // cache (ncu: 2.1 no_instruction stalls per issue).  See kWideUnroll.
    uint64_t y[P], ye[P];
#pragma unroll kWideUnroll
    for (uint32_t s = 0; s < L; ++s) {
      if (s) {
        const int b = __ffs(s) - 1;
        const bool minus = (b == k - 1) ? lane_minus : ((s >> (b + 1)) & 1);
        const uint64_t* col = (minus ? Wm : W2) + b * CS;
#pragma unroll
        for (int q = 0; q < P; ++q) {
#pragma unroll
          for (int j = 0; j < NS; j += 2) {
            const ulonglong2 c = *reinterpret_cast<const ulonglong2*>(col + q * NS + j);
            if constexpr (LAZY) {
              // PK_ALU_ADD: a runtime-zero third operand keeps the 64-bit add on
              // the ALU pipe (3-input IADD3 / IADD3.X; see pk_walk.cuh upd_step)
              r[q][j] += c.x + (PK_ALU_ADD ? zero : 0ull);
              if (j + 1 < N) r[q][j + 1] += c.y + (PK_ALU_ADD ? zero : 0ull);
            } else {
              upd(r[q][j], c.x, p(q));
              if (j + 1 < N) upd(r[q][j + 1], c.y, p(q));
            }
          }
        }
      }
      tree(y);
      if constexpr (LAZY) {
        if (!(s & 1)) {  // warp-uniform: rows < 4p -> < 2p
#pragma unroll
          for (int q = 0; q < P; ++q) {
            const uint64_t p2 = 2 * p(q);
#pragma unroll
            for (int j = 0; j < N; ++j)
              r[q][j] = r[q][j] >= p2 ? r[q][j] - p2 + (PK_ALU_ADD ? zero : 0ull) : r[q][j];
          }
        }
      }
      if (s & 1) {
        add_pair(ye, y);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) ye[q] = y[q];
      }
    }
  }
};

// One wide prime group per launch; modp_out holds a (lo, hi) 128-bit counter
// per prime of the fold2^-64-scaled residues.
template <int N, int P, bool LAZY>
__global__ void __launch_bounds__(kWalkThreads, min_ctas(N * P * 2))
    walk_modp64_kernel(const __grid_constant__ WalkArgs args) {
  using W_ = Modp64Walker<N, P, LAZY>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* slot = reinterpret_cast<uint64_t*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWalkWarps + warp;
  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * kWalkWarps;
  stage_modp64<N, P>(slot, static_cast<const uint64_t*>(args.a), args.mc.p64, args.m, args.algo,
                     threadIdx.x, blockDim.x);
  __syncthreads();
  W_ w;
  w.mc = &args.mc;
  w.zero = static_cast<uint64_t>(args.per_warp_slot);  // always 0 for F_p launches
  uint64_t tot[P];
#pragma unroll
  for (int q = 0; q < P; ++q) tot[q] = 0;
  for (uint64_t tl = gw; tl < args.tiles; tl += tw) {
    const uint64_t seg = ((args.tile0 + tl) << kTileBits) + lane;
    const bool active = seg < args.segs_total;
    w.walk(slot, slot + 2 * args.m * W_::CS, args.m, args.k, active ? seg : 0);
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const uint64_t pq = args.mc.p64[q];
      // acc < 2^k 4p with k <= 30, so hi < p
      uint64_t v = active ? fold128(w.acc_lo[q], w.acc_hi[q], pq, args.mc.pinv64[q]) : 0ull;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const uint64_t o = v + __shfl_xor_sync(0xffffffffu, v, off);
        v = min_u64(o, o - pq);
      }
      const uint64_t t = tot[q] + v;
      tot[q] = min_u64(t, t - pq);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
      unsigned long long* o = args.modp_out + 2 * q;
      const unsigned long long old = atomicAdd(o, static_cast<unsigned long long>(tot[q]));
      if (old + tot[q] < old) atomicAdd(o + 1, 1ull);
    }
  }
}

}  // namespace pk
