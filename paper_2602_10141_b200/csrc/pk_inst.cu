// Explicit instantiation of the templated walk kernels.
//
// Compiled several times by the Makefile with different -D settings so the
// ~200 kernels build in parallel:
//   -DPK_INST_F64 -DPK_CPLX=0|1 -DPK_C0P=0|1 -DPK_N_LO=.. -DPK_N_HI=..  fp64 real/complex,
//                 column 0 from shared memory (batched) or the kernel parameter
//   -DPK_INST_MODP -DPK_LAZY=0|1 -DPK_P=1..4 -DPK_N_LO=.. -DPK_N_HI=..  F_p, P primes per lane
//   -DPK_INST_HYBRID -DPK_PI=1 -DPK_WF=0|1 -DPK_N_LO=.. -DPK_N_HI=..  F_p, PI Montgomery +
//                 1 fp64 prime (WF: wide fp64 prime, two-product modmul)
//   -DPK_INST_WIDE -DPK_WLAZY=0|1 -DPK_P=1 -DPK_N_LO=.. -DPK_N_HI=..  F_p, wide moduli
//                 (Montgomery-64; WLAZY: rows reduced every second step, p < 2^60)
// Each object exports one registration function that stores the kernel
// addresses for N in [PK_N_LO, PK_N_HI] into the dispatch tables (pk_capi.cu).
#include <utility>

#include "pk_registry.h"
#include "pk_walk.cuh"
#include "pk_walk64.cuh"
#include "pk_walk_hybrid.cuh"

#define PK_CAT2(a, b) a##b
#define PK_CAT(a, b) PK_CAT2(a, b)

namespace pk {

#if defined(PK_INST_F64)
template <int... I>
static void fill(const void** tbl, std::integer_sequence<int, I...>) {
  ((tbl[PK_N_LO + I] = reinterpret_cast<const void*>(
        &walk_f64_kernel<PK_N_LO + I, (PK_CPLX != 0), (PK_C0P != 0)>)),
   ...);
}
void PK_CAT(PK_CAT(PK_CAT(PK_CAT(PK_CAT(register_f64_c, PK_CPLX), _p), PK_C0P), _), PK_N_LO)(
    const void** tbl) {
  fill(tbl, std::make_integer_sequence<int, PK_N_HI - PK_N_LO + 1>{});
}
#elif defined(PK_INST_MODP)
template <int... I>
static void fill(const void** tbl, std::integer_sequence<int, I...>) {
  ((tbl[PK_N_LO + I] = reinterpret_cast<const void*>(&walk_modp_kernel<PK_N_LO + I, PK_P, (PK_LAZY != 0)>)), ...);
}
void PK_CAT(PK_CAT(PK_CAT(PK_CAT(PK_CAT(register_modp_l, PK_LAZY), _p), PK_P), _), PK_N_LO)(const void** tbl) {
  fill(tbl, std::make_integer_sequence<int, PK_N_HI - PK_N_LO + 1>{});
}
#elif defined(PK_INST_HYBRID)
template <int... I>
static void fill(const void** tbl, std::integer_sequence<int, I...>) {
  ((tbl[PK_N_LO + I] = reinterpret_cast<const void*>(
        &walk_hybrid_kernel<PK_N_LO + I, PK_PI, 1, (PK_WF != 0)>)),
   ...);
}
void PK_CAT(PK_CAT(PK_CAT(PK_CAT(PK_CAT(register_hybrid_pi, PK_PI), _w), PK_WF), _), PK_N_LO)(
    const void** tbl) {
  fill(tbl, std::make_integer_sequence<int, PK_N_HI - PK_N_LO + 1>{});
}
#elif defined(PK_INST_WIDE)
template <int... I>
static void fill(const void** tbl, std::integer_sequence<int, I...>) {
  ((tbl[PK_N_LO + I] = reinterpret_cast<const void*>(
        &walk_modp64_kernel<PK_N_LO + I, PK_P, (PK_WLAZY != 0)>)),
   ...);
}
void PK_CAT(PK_CAT(PK_CAT(PK_CAT(PK_CAT(register_wide_l, PK_WLAZY), _p), PK_P), _), PK_N_LO)(
    const void** tbl) {
  fill(tbl, std::make_integer_sequence<int, PK_N_HI - PK_N_LO + 1>{});
}
#else
#error "define PK_INST_F64, PK_INST_MODP, PK_INST_HYBRID or PK_INST_WIDE"
#endif

}  // namespace pk
