// Dispatch tables for the templated walk kernels (filled by pk_inst.cu objects).
#pragma once

namespace pk {

constexpr int kMaxN = 48;  // largest state length with a register-resident kernel
// real fp64 walks go further: 64 doubles of state fit the register file (the
// paper's 54 x 54 real Glynn permanent)
constexpr int kMaxNReal = 64;
constexpr int kMaxP = 4;   // primes per lane in the F_p kernel

// N ranges compiled per object; must match the Makefile's INST_RANGES.
#define PK_FOR_EACH_RANGE(X) X(1, 16) X(17, 28) X(29, 36) X(37, 42) X(43, 48)

#define PK_DECL_F64(lo, hi)                         \
  void register_f64_c0_p0_##lo(const void** tbl); \
  void register_f64_c1_p0_##lo(const void** tbl); \
  void register_f64_c0_p1_##lo(const void** tbl); \
  void register_f64_c1_p1_##lo(const void** tbl);
#define PK_DECL_MODP1(lazy, lo)                          \
  void register_modp_l##lazy##_p1_##lo(const void** tbl); \
  void register_modp_l##lazy##_p2_##lo(const void** tbl); \
  void register_modp_l##lazy##_p3_##lo(const void** tbl); \
  void register_modp_l##lazy##_p4_##lo(const void** tbl);
#define PK_DECL_MODP(lo, hi) PK_DECL_MODP1(0, lo) PK_DECL_MODP1(1, lo)
// hybrid (Montgomery + fp64 primes) kernels exist for N in [kHybridMinN, kMaxN]
constexpr int kHybridMinN = 17;
#define PK_FOR_EACH_HYBRID_RANGE(X) X(17, 28) X(29, 36) X(37, 42) X(43, 48)
// (group_primes pairs one lazy Montgomery prime with one fp64 prime, PI = 1)
#define PK_DECL_HYBRID(lo, hi)                         \
  void register_hybrid_pi1_w0_##lo(const void** tbl); \
  void register_hybrid_pi1_w1_##lo(const void** tbl);
PK_FOR_EACH_HYBRID_RANGE(PK_DECL_HYBRID)
#undef PK_DECL_HYBRID
// wide (2^31 <= p < 2^62, Montgomery-64) kernels: one prime per lane (two per
// lane measured 20-30 % slower per prime: register pressure, profiles/r1_modp_rates_wide2.json)
#ifndef PK_WIDE_PMAX
#define PK_WIDE_PMAX 1  // experiment switch: 2 moduli per lane (variant builds)
#endif
constexpr int kMaxPWide = PK_WIDE_PMAX;
#if PK_WIDE_PMAX >= 2
void register_wide_l1_p2_29(const void** tbl);  // N = 29..36, p < 2^60
#endif
#define PK_DECL_WIDE1(lo, hi)                     \
  void register_wide_l0_p1_##lo(const void** tbl); \
  void register_wide_l1_p1_##lo(const void** tbl);
PK_FOR_EACH_RANGE(PK_DECL_WIDE1)
#undef PK_DECL_WIDE1
PK_FOR_EACH_RANGE(PK_DECL_F64)
void register_f64_c0_p0_49(const void** tbl);  // real, N = 49..64
void register_f64_c0_p1_49(const void** tbl);
PK_FOR_EACH_RANGE(PK_DECL_MODP)
#undef PK_DECL_F64
#undef PK_DECL_MODP
#undef PK_DECL_MODP1

}  // namespace pk
