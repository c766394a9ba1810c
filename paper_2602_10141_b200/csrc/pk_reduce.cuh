// Deterministic, device-count independent reduction of fp64 tile partials.
//
// Tiles of one matrix are grouped by GLOBAL index into groups of c tiles
// (c = max(1, tiles_total / kMaxGroups), a power of two fixed by n, never by
// the device count).  Two launches: fold_groups_kernel (one thread per group,
// many CTAs) and tree_groups_kernel (one CTA per matrix).  A group is a left fold of pair_combine; groups are then
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

constexpr int kMaxGroups = 4096;   // groups per matrix and launch (see make_plan)
constexpr int kFoldThreads = 128;
constexpr int kTreeThreads = 512;
constexpr int kRegLevels = 3;      // tree levels combined in registers (8 groups per thread)
constexpr int kPartialStride = 5;  // s_re, c_re, s_im, c_im, abs

struct Node5 {
  Pair re, im;
  double ab;
};

__device__ __forceinline__ Node5 node_combine(const Node5& a, const Node5& b) {
  return Node5{pair_combine(a.re, b.re), pair_combine(a.im, b.im), a.ab + b.ab};
}

__device__ __forceinline__ Node5 load_node(const double* q) {
  return Node5{Pair{q[0], q[1]}, Pair{q[2], q[3]}, q[4]};
}

__device__ __forceinline__ void store_node(double* q, const Node5& v) {
  q[0] = v.re.s;
  q[1] = v.re.c;
  q[2] = v.im.s;
  q[3] = v.im.c;
  q[4] = v.ab;
}

// Stage 1: left fold of each group of c tiles (one thread per group).
// partials: [B][tiles][5] for global tiles [tile0, tile0 + tiles);
// groups:   [B][ng][5] for global groups [g0, g0 + ng).
__global__ void __launch_bounds__(kFoldThreads) fold_groups_kernel(
    const double* __restrict__ partials, uint64_t tile0, uint64_t tiles, uint64_t c, uint64_t g0,
    int ng, double* __restrict__ groups) {
  const int b = blockIdx.y;
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= ng) return;
  const double* P = partials + static_cast<uint64_t>(b) * tiles * kPartialStride;
  const uint64_t lo = max((g0 + gi) * c, tile0), hi = min((g0 + gi + 1) * c, tile0 + tiles);
  Node5 acc = load_node(P + (lo - tile0) * kPartialStride);
#pragma unroll 4
  for (uint64_t t = lo + 1; t < hi; ++t) acc = node_combine(acc, load_node(P + (t - tile0) * kPartialStride));
  store_node(groups + (static_cast<uint64_t>(b) * ng + gi) * kPartialStride, acc);
}

// Stage 2: binary tree over the groups on GLOBAL indices (level L node j covers
// groups [j 2^L, (j+1) 2^L)); missing children pass their sibling through.  The
// first kRegLevels levels are combined in registers, the rest in shared memory.
// G: the ng group nodes of global groups [g0, g0 + ng); one CTA.
__device__ __forceinline__ void tree_groups_body(const double* __restrict__ G, uint64_t g0, int ng,
                                                 double* __restrict__ out) {
  constexpr int kLeaves = 1 << kRegLevels;
  __shared__ Node5 buf[2][kMaxGroups / kLeaves + 2];
  const uint64_t g1 = g0 + ng;  // exclusive
  uint64_t lo_prev = g0 >> kRegLevels, hi_prev = (g1 - 1) >> kRegLevels;
  const int cnt0 = static_cast<int>(hi_prev - lo_prev + 1);
  for (int t = threadIdx.x; t < cnt0; t += blockDim.x) {
    const uint64_t j = lo_prev + t;
    Node5 v[kLeaves];
    bool has[kLeaves];
#pragma unroll
    for (int e = 0; e < kLeaves; ++e) {
      const uint64_t g = j * kLeaves + e;
      has[e] = g >= g0 && g < g1;
      if (has[e]) v[e] = load_node(G + (g - g0) * kPartialStride);
    }
#pragma unroll
    for (int w = 1; w < kLeaves; w *= 2)
#pragma unroll
      for (int e = 0; e + w < kLeaves; e += 2 * w) {
        if (has[e] && has[e + w])
          v[e] = node_combine(v[e], v[e + w]);
        else if (has[e + w])
          v[e] = v[e + w];
        has[e] = has[e] || has[e + w];
      }
    buf[0][t] = v[0];
  }
  __syncthreads();
  int cur = 0;
  while (lo_prev != hi_prev) {
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
  if (threadIdx.x == 0) store_node(out, buf[cur][0]);
}

// One CTA per matrix b: groups [b][ng] of global groups [g0, g0 + ng).
__global__ void __launch_bounds__(kTreeThreads) tree_groups_kernel(const double* __restrict__ groups,
                                                                    uint64_t g0, int ng,
                                                                    double* __restrict__ out) {
  const int b = blockIdx.x;
  tree_groups_body(groups + static_cast<uint64_t>(b) * ng * kPartialStride, g0, ng,
                   out + static_cast<uint64_t>(b) * kPartialStride);
}

// ---------------------------------------------------------------------------
// Segmented forms for a caller's block plan (pk_ryser_f64_plan): one launch
// reduces every block's own tile range with exactly the groups and tree a
// single-range call on that block would use, so each block's root is
// bit-identical to pk_ryser_f64 on the block.
//
// Fold task i: global tiles [lo_i, hi_i), whose partials sit at consecutive
// indices from pidx_i -> group node i (a left fold, as fold_groups_kernel).
struct FoldTask {
  uint64_t lo, hi, pidx;
};
__global__ void __launch_bounds__(kFoldThreads) fold_tasks_kernel(
    const double* __restrict__ partials, const FoldTask* __restrict__ tasks, int ntasks,
    double* __restrict__ groups) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntasks) return;
  const FoldTask t = tasks[i];
  const double* P = partials + t.pidx * kPartialStride;
  Node5 acc = load_node(P);
  for (uint64_t x = 1; x < t.hi - t.lo; ++x) acc = node_combine(acc, load_node(P + x * kPartialStride));
  store_node(groups + static_cast<uint64_t>(i) * kPartialStride, acc);
}

// Tree of block b: its groups are nodes [first_b, first_b + ng_b) of `groups`,
// global group indices [g0_b, g0_b + ng_b).
struct TreeTask {
  uint64_t g0;
  int first, ng;
};
__global__ void __launch_bounds__(kTreeThreads) tree_tasks_kernel(const double* __restrict__ groups,
                                                                   const TreeTask* __restrict__ tasks,
                                                                   double* __restrict__ out) {
  const TreeTask t = tasks[blockIdx.x];
  tree_groups_body(groups + static_cast<uint64_t>(t.first) * kPartialStride, t.g0, t.ng,
                   out + static_cast<uint64_t>(blockIdx.x) * kPartialStride);
}

}  // namespace pk
