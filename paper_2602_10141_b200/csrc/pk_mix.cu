// Instruction-mix ceilings of the walk kernels, measured in-run (roofline
// denominators beside the single-pipe peaks of pk_peaks.cu).
//
// A walk's hot loop is its walker's step (flip + product tree) plus the Gray
// bookkeeping (ctz, direction, column address) and a segment restart every
// 2^k steps.  These kernels run the PRODUCTION walker structs (F64Walker,
// ModpWalker + FpPart) on one column pair held in shared memory, flipping it
// in and out, with none of the bookkeeping and no restarts, at the walk's own
// occupancy.  Their rate is the ceiling of the walk's arithmetic mix on this
// SM -- register-bank conflicts, dispatch limits and the two-pipe balance
// included -- so walk rate / mix rate is the share the Gray bookkeeping and
// the restarts cost.  (tools/micro/hybrid_mix.cu is the stand-alone form.)
//
// Units: row updates (fp64) or prime-row updates (F_p), the unit of
// SURVEY.md 8(d3).  Output per mix: units/s, units per SM clock (clock64
// spans), mean SM MHz.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <vector>

#include "pk_common.cuh"
#include "pk_walk.cuh"
#include "pk_walk_hybrid.cuh"

namespace pk {
namespace {

constexpr int kMixCols = 8;  // columns in rotation (shared memory)

struct MixOut {
  long long t0, t1, smid;
};

__device__ __forceinline__ void mix_span(long long t0, MixOut* spans) {
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    spans[blockIdx.x] = MixOut{t0, t1, smid};
  }
}

// complex fp64: the FP64 work of the walk's step pair -- n fma(+-1) row flips
// and the production product tree (F64Walker::tree) per step, the pair
// difference and its Neumaier step (F64Walker::add_pair) -- with the column in
// registers: the ceiling of the arithmetic mix itself, without the column
// loads (round 1's tools/micro/fp64_mix.cu measured 88 % of the DFMA peak for
// the same mix without the Neumaier step).
template <int N>
__global__ void __launch_bounds__(kWalkThreads, min_ctas(N * 4))
    mix_complex_kernel(const __grid_constant__ WalkArgs args, int pairs, double* sink,
                       MixOut* spans) {
  using W_ = F64Walker<N, true, false>;
  using T = double2;
  W_ w;
  w.want_abs = false;
  T c[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    w.r[j] = make_double2(0.9 + 1e-3 * j + 1e-6 * threadIdx.x, 0.1);
    c[j] = make_double2(1e-3 * j, 2e-3);
  }
  w.s_re = w.c_re = w.s_im = w.c_im = w.abs_acc = 0.0;
  const long long t0 = clock64();
  for (int e = 0; e < pairs; ++e) {
    const double sg = (e & 1) ? -1.0 : 1.0;  // add, then remove: the state stays bounded
#pragma unroll
    for (int j = 0; j < N; ++j) fma_upd(w.r[j], sg, c[j]);
    const T pe = w.tree();
#pragma unroll
    for (int j = 0; j < N; ++j) fma_upd(w.r[j], -sg, c[j]);
    const T po = w.tree();
    w.add_pair(pe, po);
  }
  mix_span(t0, spans);
  if (w.s_re == 1.2345) sink[threadIdx.x] = w.s_re + w.c_im;
}

// hybrid F_p: one lazy Montgomery prime + one fp64 prime, exactly the
// HybridWalker step (ModpWalker::step, FpPart::flip / product) and pair.
template <int N, bool WF>
__global__ void __launch_bounds__(kWalkThreads, PK_HYB_MINCTA)
    mix_hybrid_kernel(const __grid_constant__ WalkArgs args, int pairs,
                      unsigned long long* sink, MixOut* spans) {
  constexpr int NS4 = col_stride(N, 4), NS8 = col_stride(N, 8);
  __shared__ __align__(16) uint32_t cm[2][kMixCols][NS4];
  __shared__ __align__(16) double cf[2][kMixCols][NS8];
  const uint32_t p = args.mc.p[0];
  const double fp = args.mc.fp[0];
  for (int j = threadIdx.x; j < kMixCols * NS4; j += blockDim.x) {
    const uint32_t v = (j % NS4) < N ? (977u * j + 5u) % p : 0u;
    cm[0][0][j] = v;
    cm[1][0][j] = 0u - v;  // the lazy minus copy
  }
  for (int j = threadIdx.x; j < kMixCols * NS8; j += blockDim.x) {
    const double v =
        (j % NS8) < N ? static_cast<double>((1543ull * j + 3ull) % static_cast<uint64_t>(fp)) : 0.0;
    cf[0][0][j] = v;
    cf[1][0][j] = -v;
  }
  __syncthreads();
  ModpWalker<N, 1, true> mw;
  FpPart<N, 1, WF> fw;
  mw.mc = &args.mc;
  fw.mc = &args.mc;
  for (int j = 0; j < N; ++j) {
    mw.r[0][j] = (threadIdx.x * 7u + 13u * j) % p;
    fw.x[0][j] = static_cast<double>((threadIdx.x * 11ull + 17ull * j) % static_cast<uint64_t>(fp));
  }
  mw.acc[0] = 0;
  fw.acc[0] = 0.0;
  uint32_t ye[1], yo[1];
  double fe[1], fo[1];
  const long long t0 = clock64();
#pragma unroll 1
  for (int e = 0; e < pairs; ++e) {
    const int d = e & 1;  // two adds, then two removes (of different columns)
    const int b = (__ffs(e >> 1) - 1) & (kMixCols - 1);
    mw.step(cm[d][b], ye);
    fw.flip(cf[d][b]);
    fw.product(fe);
    mw.step(cm[d][(b + 1) & (kMixCols - 1)], yo);
    fw.flip(cf[d][(b + 1) & (kMixCols - 1)]);
    fw.product(fo);
    mw.add_pair(ye, yo);
    fw.acc[0] += fe[0] - fo[0];
    if constexpr (WF) fw.acc[0] = fw.reduce(fw.acc[0], 0);
  }
  mix_span(t0, spans);
  if (mw.acc[0] == 0x123456789ull && fw.acc[0] == 1.5) sink[threadIdx.x] = mw.acc[0];
}

template <class K>
int run_mix(K kernel, WalkArgs& args, int pairs, double units_per_pair_thread, double* ops_per_s,
            double* per_clk_sm, double* mhz) {
  int dev = 0, sms = 0, occ = 0;
  PK_CUDA(cudaGetDevice(&dev));
  PK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kWalkThreads, 0));
  const int grid = sms * occ;
  void* sink = nullptr;
  MixOut* spans = nullptr;
  PK_CUDA(cudaMalloc(&sink, 8 * kWalkThreads));
  PK_CUDA(cudaMalloc(&spans, sizeof(MixOut) * grid));
  cudaEvent_t e0, e1;
  PK_CUDA(cudaEventCreate(&e0));
  PK_CUDA(cudaEventCreate(&e1));
  int warm = pairs / 8;
  void* wargs[] = {&args, &warm, &sink, &spans};
  PK_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(kWalkThreads),
                           wargs, 0, nullptr));
  PK_CUDA(cudaGetLastError());
  PK_CUDA(cudaEventRecord(e0));
  void* kargs[] = {&args, &pairs, &sink, &spans};
  PK_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(kWalkThreads),
                           kargs, 0, nullptr));
  PK_CUDA(cudaEventRecord(e1));
  PK_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  PK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  std::vector<MixOut> h(grid);
  PK_CUDA(cudaMemcpy(h.data(), spans, sizeof(MixOut) * grid, cudaMemcpyDeviceToHost));
  std::vector<long long> lo(1024, LLONG_MAX), hi(1024, LLONG_MIN);
  std::vector<int> cnt(1024, 0);
  for (const MixOut& o : h) {
    const int s = static_cast<int>(o.smid) & 1023;
    lo[s] = std::min(lo[s], o.t0);
    hi[s] = std::max(hi[s], o.t1);
    cnt[s]++;
  }
  const double units_cta = units_per_pair_thread * pairs * kWalkThreads;
  double rate = 0, span = 0;
  int nsm = 0;
  for (int s = 0; s < 1024; ++s) {
    if (!cnt[s]) continue;
    rate += units_cta * cnt[s] / double(hi[s] - lo[s]);
    span += double(hi[s] - lo[s]);
    ++nsm;
  }
  *ops_per_s = units_cta * grid / (ms * 1e-3);
  *per_clk_sm = rate / nsm;
  *mhz = (span / nsm) / (ms * 1e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaFree(spans);
  return 0;
}

}  // namespace
}  // namespace pk

// out[3 i ..] = {units/s, units per SM clock, SM MHz} for the mixes named by
// pk_mix_names(); returns the count.
extern "C" int pk_measure_mix_ceilings(int device, double* out, int max_out) {
  using namespace pk;
  return pk_guard([&]() -> int {
    PK_CUDA(cudaSetDevice(device));
    WalkArgs args{};
    for (int i = 0; i < 2 * 48; ++i) args.col0[i] = 1e-3 * (i + 1) * ((i & 1) ? -1.0 : 1.0);
    // the n = 36 GPU basis's lazy and wide fp64 primes; a narrow fp64 prime
    const uint32_t p = 59652289u;
    args.mc.p[0] = p;
    args.mc.mneg[0] = mont_neg_inv32(p);
    args.mc.kneg[0] = p * ((1u << 30) / p + 2u);
    int k = 0;
    auto put = [&](double a, double b, double c) {
      if (k + 3 <= max_out) {
        out[k] = a;
        out[k + 1] = b;
        out[k + 2] = c;
      }
      k += 3;
    };
    double a, b, c;
    const int pairs = 1024;
    if (int rc = run_mix(mix_complex_kernel<32>, args, pairs, 2.0 * 32, &a, &b, &c)) return rc;
    put(a, b, c);
    args.mc.fp[0] = 868749928021.0;
    args.mc.fpinv[0] = 1.0 / args.mc.fp[0];
    if (int rc = run_mix(mix_hybrid_kernel<36, true>, args, pairs, 2.0 * 2 * 36, &a, &b, &c))
      return rc;
    put(a, b, c);
    args.mc.fp[0] = 15817573.0;  // the largest fp64 prime of n = 36 (modular.prime_pool)
    args.mc.fpinv[0] = 1.0 / args.mc.fp[0];
    if (int rc = run_mix(mix_hybrid_kernel<36, false>, args, pairs, 2.0 * 2 * 36, &a, &b, &c))
      return rc;
    put(a, b, c);
    return k / 3;
  });
}

extern "C" const char* pk_mix_names(void) {
  return "complex_32,hybrid_wide_36,hybrid_36";
}
