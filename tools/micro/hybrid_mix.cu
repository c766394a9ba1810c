// Micro-benchmark: the ceiling of the hybrid F_p walk's instruction mix.
//
// walk_hybrid_kernel<N, 1 lazy Montgomery prime, 1 wide fp64 prime> does, per
// Gray step and lane: N lazy row flips (IADD3) + an N-leaf REDC tree
// (IMAD.WIDE.U32, IMAD, IMAD.HI.U32 per REDC), N fp64 row flips (DADD) + an
// N-leaf two-product modmul tree (DMUL, DFMA, DFMA, DADD, DFMA, DADD per
// modmul), and the accumulation.  This kernel runs exactly that mix, the
// columns read from shared memory (plus / minus copies, 16-byte broadcast
// loads) like the walk, but with no Gray bookkeeping and no segment starts, at
// a chosen occupancy: its rate is the practical ceiling of the mix
// on this SM (register-bank / dispatch limits included), against which the
// walk's measured rate is judged ("prove its ceiling").
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a hybrid_mix.cu -o hybrid_mix
//   ./hybrid_mix            -> one line per (N, tree|chain4, CTAs/SM)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mont(uint32_t x, uint32_t y, uint32_t p, uint32_t mneg) {
  const uint64_t t = static_cast<uint64_t>(x) * y;
  const uint32_t m = static_cast<uint32_t>(t) * mneg;
  const uint64_t u = static_cast<uint64_t>(m) * p + t;
  return static_cast<uint32_t>(u >> 32);
}

struct FpC {
  double p, pinv;
};
__device__ __forceinline__ double red(double v, const FpC& c) {
  const double S = 6755399441055744.0;
  const double q = fma(v, c.pinv, S) - S;
  return fma(-q, c.p, v);
}
__device__ __forceinline__ double mmul(double a, double y, const FpC& c) {
  const double h = a * y;
  const double l = fma(a, y, -h);
  return red(h, c) + l;
}

template <int N, bool TREE>
__device__ __forceinline__ void products(const uint32_t* r, const double* x, uint32_t p,
                                         uint32_t mneg, const FpC& c, uint32_t& ym, double& yf) {
  constexpr int LOG = 7;
  uint32_t st[LOG];
  double sf[LOG];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    uint32_t v = r[j];
    double w = x[j];
    int l = 0;
#pragma unroll
    for (; l < LOG && ((j >> l) & 1); ++l) {
      v = mont(st[l], v, p, mneg);
      if (TREE) w = mmul(sf[l], w, c);
    }
    st[l] = v;
    sf[l] = w;
  }
  uint32_t am = 0;
  double af = 0;
  bool have = false;
#pragma unroll
  for (int l = 0; l < LOG; ++l)
    if ((N >> l) & 1) {
      am = have ? mont(st[l], am, p, mneg) : st[l];
      if (TREE) af = have ? mmul(sf[l], af, c) : sf[l];
      have = true;
    }
  ym = am;
  if (TREE) {
    yf = af;
  } else {  // four chains joined by a small tree, as the round-1 kernel
    double ch[4];
#pragma unroll
    for (int i = 0; i < N; ++i) ch[i % 4] = i < 4 ? x[i] : mmul(x[i], ch[i % 4], c);
    ch[0] = mmul(ch[0], ch[1], c);
    ch[2] = mmul(ch[2], ch[3], c);
    yf = mmul(ch[0], ch[2], c);
  }
}

template <int N, bool TREE, int MINB>
__global__ void __launch_bounds__(128, MINB) mix(int steps, uint64_t* out, uint32_t p, uint32_t mneg,
                                                 double fp, double fpinv) {
  // columns in shared memory, plus and minus copies, read as 16-byte broadcast
  // loads like the walk (walk_hybrid_kernel stages W2 / Wf the same way)
  __shared__ __align__(16) uint32_t cm[2][((N + 3) / 4) * 4];
  __shared__ __align__(16) double cf[2][((N + 1) / 2) * 2];
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    cm[0][j] = (j * 977 + 5) & 0xffff;
    cm[1][j] = 0u - cm[0][j];
    cf[0][j] = static_cast<double>((j * 1543 + 3) & 0xfffff);
    cf[1][j] = -cf[0][j];
  }
  __syncthreads();
  uint32_t r[N];
  double x[N];
  const FpC c{fp, fpinv};
  for (int j = 0; j < N; ++j) {
    r[j] = (threadIdx.x * 7 + j * 13) & 0xffff;
    x[j] = static_cast<double>((threadIdx.x * 11 + j * 17) & 0xfffff);
  }
  uint64_t accm = 0;
  double accf = 0;
  for (int s = 0; s < steps; ++s) {
    const int d = (s >> 1) & 1;  // remove on every other pair of steps
    const uint32_t* colm = cm[d];
    const double* colf = cf[d];
#pragma unroll
    for (int j = 0; j + 4 <= ((N + 3) / 4) * 4; j += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(colm + j);
      if (j < N) r[j] += v.x;
      if (j + 1 < N) r[j + 1] += v.y;
      if (j + 2 < N) r[j + 2] += v.z;
      if (j + 3 < N) r[j + 3] += v.w;
    }
#pragma unroll
    for (int j = 0; j + 2 <= N; j += 2) {
      const double2 v = *reinterpret_cast<const double2*>(colf + j);
      x[j] += v.x;
      x[j + 1] += v.y;
    }
    uint32_t ym;
    double yf;
    products<N, TREE>(r, x, p, mneg, c, ym, yf);
    accm += ym;
    accf = red(accf + yf, c);
  }
  if (accm == 0x123456789ull && accf == 1.5) out[threadIdx.x] = accm;
}

template <int N, bool TREE, int MINB>
void run(int ctas_per_sm) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* o;
  cudaMalloc(&o, 1024 * 8);
  const uint32_t p = 59652289u;  // a lazy prime of the n = 36 basis
  uint32_t inv = p;
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  const double fp = 868749928021.0;  // the wide fp64 prime of the n = 36 basis
  const int steps = 4000;
  mix<N, TREE, MINB><<<sms * ctas_per_sm, 128>>>(10, o, p, 0u - inv, fp, 1.0 / fp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  mix<N, TREE, MINB><<<sms * ctas_per_sm, 128>>>(steps, o, p, 0u - inv, fp, 1.0 / fp);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, mix<N, TREE, MINB>);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mix<N, TREE, MINB>, 128, 0);
  const double upd = 2.0 * N * steps * 128.0 * sms * ctas_per_sm;  // prime-row-updates
  printf("N=%d %s ctas/sm=%d (occ %d) regs=%d local=%zu: %.4e prime-row-updates/s\n", N,
         TREE ? "tree  " : "chain4", ctas_per_sm, occ, fa.numRegs, fa.localSizeBytes,
         upd / (ms * 1e-3));
  cudaFree(o);
}

int main() {
  run<36, true, 2>(2);
  run<36, true, 3>(3);
  run<36, false, 2>(2);
  run<36, false, 3>(3);
  run<32, true, 2>(2);
  run<32, true, 3>(3);
  return 0;
}
