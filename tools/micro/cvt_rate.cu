// Throughput of the conversions a hybrid F_p kernel would need (one warp per
// SMSP x many chains): I2F.F64.U32, F2I.S64.F64.  nvcc -O3 -arch=sm_100a cvt_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(int iters, double* out, unsigned magic) {
  unsigned x[8];
  double d[8];
  for (int c = 0; c < 8; ++c) { x[c] = threadIdx.x * 13 + c; d[c] = 1.0 + c; }
  for (int it = 0; it < iters; ++it)
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) {  // I2F.F64.U32 then DADD (chain through the double)
        d[c] += (double)x[c];
        x[c] += 1u;
      } else if (OP == 1) {  // pure I2F.F64.U32 (independent)
        asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(d[c]) : "r"(x[c] + it));
      } else {  // F2I.S64.F64
        long long v;
        asm volatile("cvt.rni.s64.f64 %0, %1;" : "=l"(v) : "d"(d[c]));
        d[c] += 1.0;
        x[c] ^= (unsigned)v;
      }
    }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += d[c] + x[c];
  if (s == magic) out[threadIdx.x] = s;
}
template <int OP>
void run(const char* name, double ops_per_inner) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, 4096);
  k<OP><<<sms * 8, 256>>>(100, o, 7);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  int iters = 4000;
  k<OP><<<sms * 8, 256>>>(iters, o, 7);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = ops_per_inner * 8.0 * iters * 256.0 * sms * 8;
  printf("%-28s %.3e ops/s = %.1f per clk per SM @1.965GHz\n", name, ops / (ms * 1e-3), ops / (ms * 1e-3) / (sms * 1.965e9));
}
int main() {
  run<0>("I2F.F64.U32 + DADD pairs", 1);
  run<1>("I2F.F64.U32", 1);
  run<2>("F2I.S64.F64 (+DADD)", 1);
  return 0;
}
