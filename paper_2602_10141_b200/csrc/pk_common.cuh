// Shared host/device helpers for the permanent engine's C-ABI library.
//
// Error convention (include/permkit_gpu.h): every entry point returns 0 on
// success or a negative status; the message is kept per calling host thread
// and read with pk_last_error().  Kernels never retain caller pointers.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace pk {

enum Status : int {
  kOk = 0,
  kErrCuda = -1,
  kErrArg = -2,
  kErrLimit = -3,
  kErrInternal = -4,
};

void set_error(const std::string& msg);
const char* last_error_cstr();

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s (%d) in %s at %s:%d", cudaGetErrorString(e),
                  static_cast<int>(e), what, file, line);
    throw Error(kErrCuda, buf);
  }
}

#define PK_CUDA(call) ::pk::cuda_check((call), #call, __FILE__, __LINE__)

// Run `body` converting exceptions into (status, last_error).
template <class F>
int pk_guard(F&& body) {
  try {
    return body();
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return kErrInternal;
  } catch (...) {
    set_error("unknown exception");
    return kErrInternal;
  }
}

// ---------------------------------------------------------------------------
// Montgomery arithmetic, R = 2^32, odd p < 2^31.
//
// mont_lazy(x, y) = x * y * 2^-32 (mod p), result in [0, 2p) whenever
// x * y < 2^32 * p  (x < p and y < 2p, or x < 2^31 / n * n and y < 2p).
// Three multiply-class instructions: IMAD.WIDE.U32 (t = x*y), IMAD (m = t*(-1/p)),
// IMAD.WIDE.U32 with 64-bit addend (t + m*p), and the high word is the result.
__host__ __device__ __forceinline__ uint32_t mont_lazy(uint32_t x, uint32_t y, uint32_t p,
                                                       uint32_t mneg) {
  const uint64_t t = static_cast<uint64_t>(x) * y;
  const uint32_t m = static_cast<uint32_t>(t) * mneg;
  const uint64_t u = static_cast<uint64_t>(m) * p + t;
  return static_cast<uint32_t>(u >> 32);
}

// -p^{-1} mod 2^32 for odd p (Newton iteration on the 2-adic inverse).
__host__ __device__ inline uint32_t mont_neg_inv32(uint32_t p) {
  uint32_t inv = p;  // correct to 3 bits for odd p
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  return 0u - inv;
}

// -p^{-1} mod 2^64 for odd p.
__host__ __device__ inline uint64_t mont_neg_inv64(uint64_t p) {
  uint64_t inv = p;
  for (int i = 0; i < 6; ++i) inv *= 2ull - p * inv;
  return 0ull - inv;
}

// ---------------------------------------------------------------------------
// Error-free transformations for the fp64 paths.

struct Pair {  // Neumaier (sum, compensation) of one real component
  double s, c;
};

// TwoSum-based combination of two compensated pairs; used for every fixed-order
// tree node so the reduction is deterministic and independent of the device
// count (a device's range is an aligned subtree).
__host__ __device__ __forceinline__ Pair pair_combine(Pair a, Pair b) {
  const double s = a.s + b.s;
  const double bp = s - a.s;
  const double ap = s - bp;
  const double e = (a.s - ap) + (b.s - bp);
  return Pair{s, (a.c + b.c) + e};
}

}  // namespace pk
