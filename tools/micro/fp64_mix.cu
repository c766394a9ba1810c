// Micro-experiment: FP64 pipe utilisation of the complex Ryser step pattern at
// fixed occupancy, without shared memory.  nvcc -O3 -arch=sm_100a fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int H, int MODE>
__global__ void __launch_bounds__(128) k(int iters, double* out, double sgv) {
  double2 r[H];
  double2 c[H];
  for (int j = 0; j < H; ++j) {
    r[j] = make_double2(0.9 + 0.001 * j + threadIdx.x * 1e-6, 0.1);
    c[j] = make_double2(1e-3 * j, 2e-3);
  }
  double s = 0, cc = 0;
  for (int it = 0; it < iters; ++it) {
    double sg = (it & 1) ? -sgv : sgv;
    for (int j = 0; j < H; ++j) { r[j].x = fma(sg, c[j].x, r[j].x); r[j].y = fma(sg, c[j].y, r[j].y); }
    double2 t[H];
    for (int j = 0; j < H; ++j) t[j] = r[j];
    if (MODE == 0) {  // tree
      for (int w = 1; w < H; w *= 2)
        for (int i = 0; i + w < H; i += 2 * w) {
          double nr = fma(t[i].x, t[i + w].x, -(t[i].y * t[i + w].y));
          t[i].y = fma(t[i].x, t[i + w].y, t[i].y * t[i + w].x);
          t[i].x = nr;
        }
    } else {  // chain
      for (int i = 1; i < H; ++i) {
        double nr = fma(t[0].x, t[i].x, -(t[0].y * t[i].y));
        t[0].y = fma(t[0].x, t[i].y, t[0].y * t[i].x);
        t[0].x = nr;
      }
    }
    s += t[0].x;  // plain add (1 FP64)
    cc += t[0].y;
  }
  if (s == 12345.0) out[threadIdx.x] = s + cc;
}
template <int H, int MODE>
void run(int ctas_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, 1024 * 8);
  int iters = 20000;
  k<H, MODE><<<sms * ctas_per_sm, 128>>>(100, o, 1e-9);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<H, MODE><<<sms * ctas_per_sm, 128>>>(iters, o, 1e-9);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fp64_per_it = 2.0 * H + 4.0 * (H - 1) + 2;
  double ops = fp64_per_it * iters * 128.0 * sms * ctas_per_sm;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k<H, MODE>);
  printf("H=%d mode=%s ctas/sm=%d regs=%d: %.3e fp64 lane-ops/s (%.1f%% of 1.78e13)\n", H,
         MODE ? "chain" : "tree", ctas_per_sm, fa.numRegs, ops / (ms * 1e-3), 100 * ops / (ms * 1e-3) / 1.78e13);
  cudaFree(o);
}
// real walk mix: DFMA update + DMUL tree, H real rows per thread
template <int H>
__global__ void __launch_bounds__(128) kr(int iters, double* out, double sgv) {
  double r[H], c[H];
  for (int j = 0; j < H; ++j) {
    r[j] = 0.9 + 0.001 * j + threadIdx.x * 1e-6;
    c[j] = 1e-3 * j;
  }
  double s = 0;
  for (int it = 0; it < iters; ++it) {
    double sg = (it & 1) ? -sgv : sgv;
    for (int j = 0; j < H; ++j) r[j] = fma(sg, c[j], r[j]);
    double t[H];
    for (int j = 0; j < H; ++j) t[j] = r[j];
    for (int w = 1; w < H; w *= 2)
      for (int i = 0; i + w < H; i += 2 * w) t[i] *= t[i + w];
    s += t[0];
  }
  if (s == 12345.0) out[threadIdx.x] = s;
}
template <int H>
void runr(int ctas_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, 1024 * 8);
  int iters = 40000;
  kr<H><<<sms * ctas_per_sm, 128>>>(100, o, 1e-9);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kr<H><<<sms * ctas_per_sm, 128>>>(iters, o, 1e-9);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (2.0 * H) * iters * 128.0 * sms * ctas_per_sm;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kr<H>);
  printf("real H=%d ctas/sm=%d regs=%d: %.3e fp64 lane-ops/s (%.1f%% of 1.78e13)\n", H, ctas_per_sm,
         fa.numRegs, ops / (ms * 1e-3), 100 * ops / (ms * 1e-3) / 1.78e13);
  cudaFree(o);
}
int main() {
  runr<32>(2); runr<32>(3); runr<32>(4);
  run<16, 0>(1); run<16, 0>(2); run<16, 0>(3); run<16, 0>(4);
  run<16, 1>(2); run<16, 1>(3); run<16, 1>(4);
  run<8, 0>(4); run<8, 0>(8);
  run<32, 0>(1); run<32, 0>(2);
  return 0;
}
