// Pipe-rate micro-benchmarks for the roofline denominators.
//
// MEASURED_PEAKS.json carries only HBM and bf16 tensor figures; the Gray-code
// Ryser walk is bound by the FP64 pipe (complex/real fp64) or by the integer
// multiply (IMAD) pipe (F_p Montgomery).  These kernels measure those issue
// rates on the box in the same run as the bench: every thread keeps 8
// independent dependency chains of one instruction class so the pipe, not
// latency, is the limit.  Inline PTX pins the instruction class; the SASS
// listing in profiles/ confirms the opcode (DFMA, DADD, DMUL, IMAD,
// IMAD.WIDE.U32, IMAD.HI.U32, LOP3/IADD3).
//
// Output: lane-operations per second for the whole GPU, and lane-operations
// per SM clock (from in-kernel clock64 spans, so DVFS does not skew it).

#include <cstdint>
#include <cuda_runtime.h>

#include "pk_common.cuh"

namespace pk {
namespace {

constexpr int kChains = 8;
constexpr int kPeakThreads = 256;

enum PeakOp : int {
  kDFMA = 0,
  kDADD = 1,
  kDMUL = 2,
  kIMAD = 3,
  kIMADWIDE = 4,
  kIMADHI = 5,
  kALU = 6,
  kMONT = 7,
  kFFMA = 8,
  kNumPeakOps = 9
};

// lane-ops of the measured class per inner iteration (per thread)
__host__ __device__ constexpr int ops_per_iter(int op) {
  return op == kMONT ? 3 * kChains : kChains;  // ALU: one IADD3 per op
}

template <int OP>
__global__ void __launch_bounds__(kPeakThreads) peak_kernel(int iters, uint64_t* sink,
                                                            long long* spans, uint64_t magic) {
  long long t0 = clock64();
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t keep = 0;
  if constexpr (OP == kDFMA || OP == kDADD || OP == kDMUL) {
    double x[kChains];
    const double y = 1.0000001 + 1e-9 * (tid & 7), z = 1e-7;
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = 0.5 + c * 0.125;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if constexpr (OP == kDFMA)
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(y), "d"(z));
        else if constexpr (OP == kDADD)
          asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[c]) : "d"(z));
        else
          asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x[c]) : "d"(y));
      }
    }
    double acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc += x[c];
    keep = __double_as_longlong(acc);
  } else if constexpr (OP == kFFMA) {
    float x[kChains];
    const float y = 1.0001f + 1e-6f * (tid & 7), z = 1e-5f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = 0.5f + c * 0.125f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < kChains; ++c)
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y), "f"(z));
    }
    float acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc += x[c];
    keep = __float_as_uint(acc);
  } else if constexpr (OP == kIMADWIDE) {
    // x <- lo(x) * hi(x) (64-bit): one IMAD.WIDE.U32 per op, no extra ALU
    uint64_t x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = (static_cast<uint64_t>(tid + c) << 32) | (tid * 7u + 3u);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < kChains; ++c)
        asm volatile("{ .reg .b32 lo, hi; mov.b64 {lo, hi}, %0; mul.wide.u32 %0, lo, hi; }"
                     : "+l"(x[c]));
    }
    for (int c = 0; c < kChains; ++c) keep ^= x[c];
  } else if constexpr (OP == kMONT) {
    // the F_p kernel's lazy Montgomery step, y <- REDC(y * y) (p < 2^30 keeps it in range)
    const uint32_t p = 1073741789u;
    const uint32_t mneg = mont_neg_inv32(p);
    uint32_t y[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) y[c] = (tid * 3u + c) & 0x3fffffffu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) y[c] = mont_lazy(y[c], y[c], p, mneg);
    }
    for (int c = 0; c < kChains; ++c) keep ^= y[c];
  } else {
    // IMAD: x <- x*x + z;  IMAD.HI: x <- hi(x*x) + z;  ALU: IADD3 chains that
    // read a neighbouring chain (x_c <- x_c + x_{c+1} + z) so nothing folds
    uint32_t x[kChains];
    const uint32_t z = 0x7F4A7C15u + tid;
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = tid * 7u + c * 0x9E3779B1u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if constexpr (OP == kIMAD)
          asm volatile("mad.lo.u32 %0, %0, %0, %1;" : "+r"(x[c]) : "r"(z));
        else if constexpr (OP == kIMADHI)
          asm volatile("mad.hi.u32 %0, %0, %0, %1;" : "+r"(x[c]) : "r"(z));
        else
          asm volatile("{ add.u32 %0, %0, %1; add.u32 %0, %0, %2; }"
                       : "+r"(x[c]) : "r"(x[(c + 1) % kChains]), "r"(z));
      }
    }
    for (int c = 0; c < kChains; ++c) keep ^= x[c];
  }
  long long t1 = clock64();
  if (keep == magic) sink[tid] = keep;  // runtime value: the chains cannot be elided
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    spans[3 * blockIdx.x + 0] = t0;
    spans[3 * blockIdx.x + 1] = t1;
    spans[3 * blockIdx.x + 2] = smid;
  }
}

template <int OP>
int run_peak(int sms, int blocks_per_sm, int iters, double* ops_per_s, double* ops_per_clk_sm,
             double* mhz) {
  const int grid = sms * blocks_per_sm;
  uint64_t* sink = nullptr;
  long long* spans = nullptr;
  PK_CUDA(cudaMalloc(&sink, sizeof(uint64_t) * grid * kPeakThreads));
  PK_CUDA(cudaMalloc(&spans, sizeof(long long) * 3 * grid));
  cudaEvent_t e0, e1;
  PK_CUDA(cudaEventCreate(&e0));
  PK_CUDA(cudaEventCreate(&e1));
  peak_kernel<OP><<<grid, kPeakThreads>>>(iters / 8, sink, spans, 0x5eed5eed5eedull);  // warm-up
  PK_CUDA(cudaGetLastError());
  PK_CUDA(cudaEventRecord(e0));
  peak_kernel<OP><<<grid, kPeakThreads>>>(iters, sink, spans, 0x5eed5eed5eedull);
  PK_CUDA(cudaEventRecord(e1));
  PK_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  PK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  std::vector<long long> h(3 * grid);
  PK_CUDA(cudaMemcpy(h.data(), spans, sizeof(long long) * 3 * grid, cudaMemcpyDeviceToHost));
  // per-SM span: max end - min start over the CTAs that ran on that SM
  std::vector<long long> lo(1024, INT64_MAX), hi(1024, INT64_MIN);
  std::vector<int> cnt(1024, 0);
  for (int b = 0; b < grid; ++b) {
    int sm = static_cast<int>(h[3 * b + 2]) & 1023;
    lo[sm] = std::min(lo[sm], h[3 * b]);
    hi[sm] = std::max(hi[sm], h[3 * b + 1]);
    cnt[sm]++;
  }
  double rate_sum = 0, span_sum = 0;
  int nsm = 0;
  const double ops_per_cta = double(ops_per_iter(OP)) * iters * kPeakThreads;
  for (int s = 0; s < 1024; ++s) {
    if (!cnt[s]) continue;
    rate_sum += ops_per_cta * cnt[s] / double(hi[s] - lo[s]);
    span_sum += double(hi[s] - lo[s]);
    ++nsm;
  }
  *ops_per_s = ops_per_cta * grid / (ms * 1e-3);
  *ops_per_clk_sm = rate_sum / nsm;
  *mhz = (span_sum / nsm) / (ms * 1e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaFree(spans);
  return 0;
}


// ---------------------------------------------------------------------------
// Dependent-chain latencies (one warp per SM, one chain): cycles per op.
template <int OP>
__global__ void lat_kernel(int iters, uint64_t* sink, long long* cyc, uint64_t magic) {
  __shared__ uint32_t sm[64];
  const unsigned tid = threadIdx.x;
  if (tid < 64) sm[tid] = (tid + 1) & 63;
  __syncthreads();
  uint64_t keep = 0;
  long long t0 = clock64();
  if constexpr (OP == 0) {  // DFMA
    double x = 0.5 + tid;
    for (int i = 0; i < iters; ++i) asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(x));
    keep = __double_as_longlong(x);
  } else if constexpr (OP == 1) {  // DMUL -> DFMA pair (one complex-product link)
    double x = 0.5 + tid, y = 0.25;
    for (int i = 0; i < iters; ++i) {
      asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(y) : "d"(x));
      asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(x) : "d"(y));
    }
    keep = __double_as_longlong(x);
  } else if constexpr (OP == 2) {  // IMAD
    uint32_t x = tid + 3;
    for (int i = 0; i < iters; ++i) asm volatile("mad.lo.u32 %0, %0, %0, %0;" : "+r"(x));
    keep = x;
  } else if constexpr (OP == 3) {  // Montgomery REDC link
    uint32_t y = tid + 5;
    const uint32_t p = 1073741789u, mneg = mont_neg_inv32(p);
    for (int i = 0; i < iters; ++i) y = mont_lazy(y, y, p, mneg);
    keep = y;
  } else if constexpr (OP == 4) {  // LDS
    uint32_t x = tid & 63;
    for (int i = 0; i < iters; ++i) x = sm[x];
    keep = x;
  } else {  // SHFL
    uint32_t x = tid;
    for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1;
    keep = x;
  }
  long long t1 = clock64();
  if (keep == magic) sink[tid] = keep;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
double run_lat(int iters) {
  uint64_t* sink = nullptr;
  long long* cyc = nullptr;
  PK_CUDA(cudaMalloc(&sink, sizeof(uint64_t) * 32));
  PK_CUDA(cudaMalloc(&cyc, sizeof(long long)));
  lat_kernel<OP><<<1, 32>>>(iters / 4, sink, cyc, 0x5eedull);
  lat_kernel<OP><<<1, 32>>>(iters, sink, cyc, 0x5eedull);
  PK_CUDA(cudaGetLastError());
  long long h = 0;
  PK_CUDA(cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
  cudaFree(sink);
  cudaFree(cyc);
  return double(h) / iters;
}
}  // namespace
}  // namespace pk

extern "C" int pk_measure_peaks(int device, double* out, int max_out) {
  using namespace pk;
  return pk_guard([&]() -> int {
    PK_CUDA(cudaSetDevice(device));
    int sms = 0;
    PK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int bps = 8;  // 8 x 256 threads = 64 warps per SM
    const int iters = 4096;
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
#define PK_PEAK(OP)                                                   \
  {                                                                   \
    int rc = run_peak<OP>(sms, bps, iters, &a, &b, &c);               \
    if (rc) return rc;                                                \
    put(a, b, c);                                                     \
  }
    PK_PEAK(kDFMA) PK_PEAK(kDADD) PK_PEAK(kDMUL) PK_PEAK(kIMAD) PK_PEAK(kIMADWIDE)
    PK_PEAK(kIMADHI) PK_PEAK(kALU) PK_PEAK(kMONT) PK_PEAK(kFFMA)
#undef PK_PEAK
    return k / 3;
  });
}

extern "C" const char* pk_peak_names(void) {
  return "dfma,dadd,dmul,imad,imad_wide,imad_hi,iadd3,mont_mul_3imad,ffma";
}

extern "C" int pk_measure_latencies(int device, double* out, int max_out) {
  using namespace pk;
  return pk_guard([&]() -> int {
    PK_CUDA(cudaSetDevice(device));
    const int iters = 1 << 14;
    double v[6] = {run_lat<0>(iters), run_lat<1>(iters), run_lat<2>(iters),
                   run_lat<3>(iters), run_lat<4>(iters), run_lat<5>(iters)};
    for (int i = 0; i < 6 && i < max_out; ++i) out[i] = v[i];
    return 6;
  });
}

extern "C" const char* pk_latency_names(void) {
  return "dfma,dmul_dfma_pair,imad,mont_redc,lds,shfl";
}
