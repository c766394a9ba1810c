// Micro-experiment harness: time walk_f64_kernel<N, complex, C0P> under compile-time
// variants (-DPK_EXP_NOKAHAN, -DPK_EXP_NOLDS, -DPK_MINCTA_T=..., -DPK_EXP_SMEM_C0 for
// column 0 from shared memory instead of the kernel parameter).
//   nvcc -O3 -std=c++17 -arch=sm_100a -I../../paper_2602_10141_b200/csrc walk_exp.cu
#include <cstdio>
#include <vector>
#include "pk_walk.cuh"
namespace pk {
void set_error(const std::string&) {}
}
int main(int argc, char** argv) {
  using namespace pk;
  constexpr int N = 32;
#ifdef PK_EXP_REAL
  constexpr bool CPLX = false;
#else
  constexpr bool CPLX = true;
#endif
  const int n = N, m = N, k = 10;
  std::vector<double> a(2 * n * n);
  for (int i = 0; i < 2 * n * n; ++i) a[i] = 0.1 * ((i * 7919) % 13 - 6) / 6.0;
  double *da, *dp;
  cudaMalloc(&da, a.size() * 8);
  cudaMemcpy(da, a.data(), a.size() * 8, cudaMemcpyHostToDevice);
  const uint64_t tiles = 1ull << (m - k - 5);
  cudaMalloc(&dp, tiles * 5 * 8);
#ifdef PK_EXP_SMEM_C0
  constexpr bool C0P = false;
#else
  constexpr bool C0P = true;
#endif
  const void* fn = (const void*)&walk_f64_kernel<N, CPLX, C0P>;
  const int eb = CPLX ? 16 : 8;
  const int smem = ((C0P ? 2 : 1) * m + 1) * col_stride(n, eb) * eb;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kWalkThreads, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, fn);
  WalkArgs w{};
  w.a = da; w.B = 1; w.n = n; w.m = m; w.algo = 0; w.k = k; w.per_warp_slot = 0;
  w.tile0 = 0; w.tiles = tiles; w.segs_total = 1ull << (m - k); w.partials = dp; w.want_abs = 0;
  for (int i = 0; i < n; ++i) {  // Ryser column 0 = a[:, 0]
    if (CPLX) { w.col0[2 * i] = a[2 * (i * n)]; w.col0[2 * i + 1] = a[2 * (i * n) + 1]; }
    else w.col0[i] = a[i * n];
  }
  const int grid = sms * occ;
  void* args[] = {&w};
  cudaLaunchKernel(fn, grid, kWalkThreads, args, smem, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 3; ++it) cudaLaunchKernel(fn, grid, kWalkThreads, args, smem, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  const double R = CPLX ? 2.966e12 : 8.9e12;
  printf("%s regs=%d local=%zu occ=%d: %.2f ms  %.3e upd/s  %.3f of R(%.3e)\n", argv[0], fa.numRegs,
         fa.localSizeBytes, occ, ms, n * 2.0 * (1ull << (m - 1)) / (ms * 1e-3),
         n * 2.0 * (1ull << (m - 1)) / (ms * 1e-3) / R, R);
  return 0;
}
