// Deterministic, device-count independent reduction of fp64 tile partials.
//
// Tiles of one matrix are grouped by GLOBAL index into groups of c tiles
// (c = max(1, tiles_total / kMaxGroups), a power of two fixed by n, never by
// the device count).  A group is a left fold of pair_combine; groups are then
// combined by a binary tree whose nodes are also aligned on global indices.
// A device that owns an aligned power-of-two run of groups therefore produces
// exactly one subtree root, and combining the device roots with the same rule
// (pk_tree_combine on the host) reproduces the single-device result bit for bit.
// This keeps the reference's determinism contract (engine.py:5-8: results
// depend on the plan, never on the worker count) across 1/2/4/8 GPUs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pk_common.cuh"

namespace pk {

constexpr int kMaxGroups = 512;
constexpr int kReduceThreads = 256;
constexpr int kPartialStride = 5;  // s_re, c_re, s_im, c_im, abs

struct Node5 {
  Pair re, im;
  double ab;
};

__device__ __forceinline__ Node5 node_combine(const Node5& a, const Node5& b) {
  return Node5{pair_combine(a.re, b.re), pair_combine(a.im, b.im), a.ab + b.ab};
}

// partials: [B][tiles][5] for global tiles [tile0, tile0 + tiles); out: [B][5]
__global__ void __launch_bounds__(kReduceThreads) reduce_tiles_kernel(const double* __restrict__ partials,
                                                                      uint64_t tile0, uint64_t tiles,
                                                                      uint64_t c, double* out) {
  __shared__ Node5 buf[2][kMaxGroups + 2];
  const int b = blockIdx.x;
  const double* P = partials + static_cast<uint64_t>(b) * tiles * kPartialStride;
  const uint64_t g0 = tile0 / c, g1 = (tile0 + tiles - 1) / c + 1;
  const int ng = static_cast<int>(g1 - g0);
  for (int gi = threadIdx.x; gi < ng; gi += blockDim.x) {
    const uint64_t lo = max((g0 + gi) * c, tile0), hi = min((g0 + gi + 1) * c, tile0 + tiles);
    Node5 acc{};
    bool first = true;
    for (uint64_t t = lo; t < hi; ++t) {
      const double* q = P + (t - tile0) * kPartialStride;
      const Node5 v{Pair{q[0], q[1]}, Pair{q[2], q[3]}, q[4]};
      acc = first ? v : node_combine(acc, v);
      first = false;
    }
    buf[0][gi] = acc;
  }
  __syncthreads();
  // binary tree on global indices: level L node j covers groups [j 2^L, (j+1) 2^L)
  int cur = 0;
  uint64_t lo_prev = g0, hi_prev = g1 - 1;  // inclusive node index range at level L-1
  for (int L = 1; lo_prev != hi_prev; ++L) {
    const uint64_t lo = lo_prev >> 1, hi = hi_prev >> 1;
    const int cnt = static_cast<int>(hi - lo + 1);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const uint64_t j = lo + t;
      const uint64_t l = 2 * j, r = 2 * j + 1;
      const bool hl = l >= lo_prev && l <= hi_prev, hr = r >= lo_prev && r <= hi_prev;
      Node5 v;
      if (hl && hr)
        v = node_combine(buf[cur][l - lo_prev], buf[cur][r - lo_prev]);
      else if (hl)
        v = buf[cur][l - lo_prev];
      else
        v = buf[cur][r - lo_prev];
      buf[cur ^ 1][t] = v;
    }
    __syncthreads();
    cur ^= 1;
    lo_prev = lo;
    hi_prev = hi;
  }
  if (threadIdx.x == 0) {
    const Node5 v = buf[cur][0];
    double* o = out + static_cast<uint64_t>(b) * kPartialStride;
    o[0] = v.re.s;
    o[1] = v.re.c;
    o[2] = v.im.s;
    o[3] = v.im.c;
    o[4] = v.ab;
  }
}

}  // namespace pk
