// Host orchestration and the extern "C" boundary (include/permkit_gpu.h).
//
// Replaces, for the GPU build, the execution half of the reference engine:
//   engine._run_plan's fast branches (reference engine.py:213-258): per-block
//     numba calls on a ThreadPoolExecutor + ordered Kahan combine
//   the per-sample / per-t / per-prime pools of ensembles.sample_permanents
//     (ensembles.py:142-158), geodesics.sweep (geodesics.py:153-179) and
//     modular.schur_permanent_exact (modular.py:188-206)
// with: one host thread per GPU, a persistent walk kernel per device, a
// deterministic device-side tree reduction, and a host combine of <= 8 roots.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>

#include "../../include/permkit_gpu.h"
#include "pk_block.cuh"
#include "pk_common.cuh"
#include "pk_reduce.cuh"
#include "pk_registry.h"
#include "pk_walk.cuh"
#include "pk_walk_hybrid.cuh"

namespace pk {

// ---------------------------------------------------------------------------
// errors

namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }

#define PK_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) fail((code), (msg)); \
  } while (0)

// ---------------------------------------------------------------------------
// kernel tables

struct Tables {
  const void* f64[2][2][kMaxNReal + 1] = {};      // [cplx][column 0 in param][N]; N > 48: real
  const void* modp[2][kMaxP + 1][kMaxN + 1] = {};  // [lazy][P][N]
  const void* hybrid[2][kMaxN + 1] = {};            // [wide fp][N]: 1 lazy + 1 fp64 prime
  const void* wide[2][kMaxPWide + 1][kMaxN + 1] = {};  // [lazy][P][N], Montgomery-64
};

static const Tables& tables() {
  static const Tables t = [] {
    Tables t;
#define PK_REG(lo, hi)                       \
  register_f64_c0_p0_##lo(t.f64[0][0]);      \
  register_f64_c1_p0_##lo(t.f64[1][0]);      \
  register_f64_c0_p1_##lo(t.f64[0][1]);      \
  register_f64_c1_p1_##lo(t.f64[1][1]);      \
  register_modp_l0_p1_##lo(t.modp[0][1]);   \
  register_modp_l0_p2_##lo(t.modp[0][2]);   \
  register_modp_l0_p3_##lo(t.modp[0][3]);   \
  register_modp_l0_p4_##lo(t.modp[0][4]);   \
  register_modp_l1_p1_##lo(t.modp[1][1]);   \
  register_modp_l1_p2_##lo(t.modp[1][2]);   \
  register_modp_l1_p3_##lo(t.modp[1][3]);   \
  register_modp_l1_p4_##lo(t.modp[1][4]);
    PK_FOR_EACH_RANGE(PK_REG)
#undef PK_REG
    register_f64_c0_p0_49(t.f64[0][0]);
    register_f64_c0_p1_49(t.f64[0][1]);
#define PK_REGH(lo, hi)                         \
  register_hybrid_pi1_w0_##lo(t.hybrid[0]);    \
  register_hybrid_pi1_w1_##lo(t.hybrid[1]);
    PK_FOR_EACH_HYBRID_RANGE(PK_REGH)
#undef PK_REGH
#define PK_REGW1(lo, hi)                 \
  register_wide_l0_p1_##lo(t.wide[0][1]); \
  register_wide_l1_p1_##lo(t.wide[1][1]);
    PK_FOR_EACH_RANGE(PK_REGW1)
#undef PK_REGW1
#if PK_WIDE_PMAX >= 2
    register_wide_l1_p2_29(t.wide[1][2]);
#endif
    return t;
  }();
  return t;
}

// ---------------------------------------------------------------------------
// per-device context

struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) PK_CUDA(cudaFree(p));
      p = nullptr;
      cap = 0;
      PK_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
      cap = std::max<size_t>(bytes, 256);
    }
    return p;
  }
};

struct DevCtx {
  int dev = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  DBuf a, partials, groups, out, primes, starts, lens, blockout, blockabs, modp_out;
  std::map<std::pair<const void*, int>, int> occ;  // (kernel, smem) -> CTAs per SM
  // per-matrix batched walks: launches round-robin over kAux streams so each
  // launch's tail overlaps the next launch (created on first use)
  static constexpr int kAux = 16;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t ev_main = nullptr, ev_aux[kAux] = {};
  void ensure_aux() {
    if (aux[0]) return;
    for (int i = 0; i < kAux; ++i) {
      PK_CUDA(cudaStreamCreateWithFlags(&aux[i], cudaStreamNonBlocking));
      PK_CUDA(cudaEventCreateWithFlags(&ev_aux[i], cudaEventDisableTiming));
    }
    PK_CUDA(cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming));
  }
};

static std::mutex g_ctx_mu;
static DevCtx* g_ctx[64] = {};

static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

static int physical_device_count() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    return 0;
  }
  PK_CUDA(e);
  return n;
}

// $PK_LOGICAL_DEVICES = L > 0 (test and measurement hook): the library reports
// L devices and maps logical device d onto physical GPU d mod (visible GPUs),
// each with its own context (stream, buffers, lock, host thread).  Every
// multi-device code path -- the per-device host threads, the range and modulus
// splits and the combine of the device results -- then runs on a one-GPU box
// exactly as it does on eight GPUs (the devices never wait on each other).
// pk_set_logical_devices() changes it at run time; a context, once created,
// keeps its GPU, and logical d < (visible GPUs) is GPU d in both modes.
static std::atomic<int> g_logical{-1};
static int logical_devices() {
  int L = g_logical.load();
  if (L < 0) {
    L = std::clamp(env_int("PK_LOGICAL_DEVICES", 0), 0, 64);
    g_logical.store(L);
  }
  return L;
}

static int device_count() {
  const int nd = physical_device_count();
  return (nd > 0 && logical_devices() > 0) ? logical_devices() : nd;
}

// Logical device d of every entry point is device base + d, so that one
// process per GPU (torchrun) can address "its" GPU as device 0.
static std::atomic<int> g_device_base{0};

static DevCtx& ctx(int logical) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  const int idx = logical + g_device_base.load();
  PK_REQUIRE(logical >= 0 && idx < 64, kErrArg, "device index out of range");
  if (!g_ctx[idx]) {
    const int nphys = physical_device_count();
    const int nd = device_count();
    PK_REQUIRE(idx < nd, kErrArg,
               "CUDA device " + std::to_string(idx) + " not available (" + std::to_string(nd) +
                   " visible)");
    const int dev = logical_devices() > 0 ? idx % nphys : idx;
    auto* c = new DevCtx;
    c->dev = dev;
    PK_CUDA(cudaSetDevice(dev));
    PK_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev));
    PK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    g_ctx[idx] = c;
  }
  return *g_ctx[idx];
}

static int occupancy(DevCtx& c, const void* fn, int threads, int smem) {
  auto key = std::make_pair(fn, smem);
  auto it = c.occ.find(key);
  if (it != c.occ.end()) return it->second;
  if (smem > 48 * 1024) {
    PK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  int nb = 0;
  PK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem));
  PK_REQUIRE(nb > 0, kErrLimit,
             "walk kernel does not fit on an SM (shared memory " + std::to_string(smem) + " B)");
  c.occ[key] = nb;
  return nb;
}

// ---------------------------------------------------------------------------
// plans

// Ragged ends of unaligned ranges are walked by the exact kernel (one thread per
// piece, a serial chain: ~0.5-1 us per step), in aligned pieces of <= 2^6
// indices so that many short pieces run in parallel.
constexpr int kPieceBits = 6;

struct Plan {
  int n = 0, m = 0, k = 0;   // k = 0: no aligned tiles (tiny m), everything ragged
  uint64_t tiles_total = 0;  // aligned tiles per matrix over the whole range
  uint64_t group = 1;        // tiles per reduction group (global alignment)
  int piece_bits = 10;       // ragged pieces are aligned to 2^piece_bits
};

// The plan depends on (n, algo) only -- never on a batch size, a device count
// or a chunking -- so a matrix's fp64 bits are the same whichever call walks it
// (single, batched, split over devices; reference engine.py:5-8).
static Plan make_plan(int n, int algo) {
  Plan p;
  p.n = n;
  p.m = algo == PK_ALGO_RYSER ? n : n - 1;
  const int m = p.m;
  if (m < 6) {
    p.k = 0;
    p.piece_bits = std::max(m, 1);
    return p;
  }
  // tiles of 2^kTileBits segments of 2^k indices; ~2^17 tiles per matrix
  const int kmin = std::min(m - kTileBits, 8);
  p.k = std::max(kmin, m - kTileBits - 17);
  // test / measurement hook ($PK_PLAN_K, read per call): force the segment
  // bits, e.g. so that a tile of an n > 48 walk (2^(m - 17) indices per lane
  // by default) is short enough for an oracle comparison or a rate sample
  if (const int kf = env_int("PK_PLAN_K", 0); kf > 0) p.k = std::clamp(kf, 1, m - kTileBits);
  p.tiles_total = 1ull << (m - p.k - kTileBits);
  p.group = std::max<uint64_t>(1, p.tiles_total / kMaxGroups);
  p.piece_bits = std::min(p.k, kPieceBits);
  return p;
}

// Batched walks with one single-matrix (column 0 in the parameter) launch per
// matrix: <= 2^10 tiles per matrix, independent of the batch size.  Used when a
// matrix is large enough (m >= kPerMatrixMinM) that a launch is a useful amount
// of work; $PK_BATCH_PER_MATRIX=0/1 forces either mode (measurement).
// complex launches are ~3x longer than real ones at the same m (6 vs 2 FP64
// instructions per row update), so real walks switch later
constexpr int kPerMatrixMinM = 20, kPerMatrixMinMReal = 21;
static Plan make_plan_per_matrix(int n, int algo) {
  Plan p = make_plan(n, algo);
  if (p.k == 0) return p;
  const int kmin = std::min(p.m - kTileBits, 8);
  p.k = std::max(kmin, p.m - kTileBits - 10);
  p.tiles_total = 1ull << (p.m - p.k - kTileBits);
  p.group = std::max<uint64_t>(1, p.tiles_total / kMaxGroups);
  p.piece_bits = std::min(p.k, kPieceBits);
  return p;
}
static bool batch_per_matrix(int m, bool cplx) {
  static const int force = env_int("PK_BATCH_PER_MATRIX", -1);
  return force >= 0 ? force != 0 : m >= (cplx ? kPerMatrixMinM : kPerMatrixMinMReal);
}
// test hook: cap the matrices per sub-batch ($PK_BATCH_SUBBATCH) so small tests
// exercise the sub-batch loops (buffer reuse across sub-batches)
static int subbatch_cap(int sb) {
  const int cap = env_int("PK_BATCH_SUBBATCH", 0);  // read per call (tests set it)
  return cap > 0 ? std::min(sb, cap) : sb;
}
// streams the per-matrix launches rotate over ($PK_BATCH_STREAMS, measurement)
static int batch_streams() {
  static const int ns = std::clamp(env_int("PK_BATCH_STREAMS", 16), 1, DevCtx::kAux);
  return ns;
}

struct Range {
  uint64_t start, end;         // [start, end)
  uint64_t t0 = 0, t1 = 0;     // aligned tiles [t0, t1)
  std::vector<std::pair<uint64_t, uint64_t>> head, tail;  // (start, len) pieces
};

static void split_pieces(uint64_t s, uint64_t e, int bits,
                         std::vector<std::pair<uint64_t, uint64_t>>& out) {
  const uint64_t span = 1ull << bits;
  while (s < e) {
    const uint64_t nxt = std::min(e, (s / span + 1) * span);
    out.emplace_back(s, nxt - s);
    s = nxt;
  }
}

static Range make_range(const Plan& p, uint64_t start, uint64_t length) {
  Range r;
  r.start = start;
  r.end = start + length;
  if (length == 0) return r;
  if (p.k == 0) {
    split_pieces(r.start, r.end, p.piece_bits, r.head);
    return r;
  }
  const int tb = p.k + kTileBits;
  const uint64_t ts = 1ull << tb;
  const uint64_t A = (start + ts - 1) / ts * ts, Bt = r.end / ts * ts;
  if (A < Bt) {
    r.t0 = A >> tb;
    r.t1 = Bt >> tb;
    split_pieces(r.start, A, p.piece_bits, r.head);
    split_pieces(Bt, r.end, p.piece_bits, r.tail);
  } else {
    split_pieces(r.start, r.end, p.piece_bits, r.head);
  }
  return r;
}

// ---------------------------------------------------------------------------
// fp64 device work

struct Node {
  Pair re{0, 0}, im{0, 0};
  double ab = 0;
};
static Node node_combine_h(const Node& a, const Node& b) {
  return Node{pair_combine(a.re, b.re), pair_combine(a.im, b.im), a.ab + b.ab};
}
static Node node_from5(const double* v) { return Node{Pair{v[0], v[1]}, Pair{v[2], v[3]}, v[4]}; }

// Enqueue walk + reduce for matrices already on the device.  Returns the
// number of kernel launches.  d_out receives [B][5] roots.
struct F64Launch {
  const void* fn;
  int grid, smem, per_warp, occ;
  WalkArgs args;
};

// h_a: the host copy of a single matrix (B == 1).  When given, walk column 0
// goes into the kernel parameter (WalkArgs::col0) and the C0P kernel runs.
static F64Launch prepare_f64(DevCtx& c, const Plan& p, bool cplx, int algo, int B,
                             const double* d_a, uint64_t t0, uint64_t nt, bool want_abs,
                             double* d_partials, const double* h_a = nullptr) {
  const int nmax = cplx ? kMaxN : kMaxNReal;
  PK_REQUIRE(p.n >= 1 && p.n <= nmax, kErrLimit,
             "dimension " + std::to_string(p.n) + " exceeds the GPU kernel range n <= " +
                 std::to_string(nmax) + (cplx ? " (complex)" : " (real)"));
  static_assert(sizeof(WalkArgs::col0) / sizeof(double) >= 2 * kMaxN, "col0 too small");
  static_assert(sizeof(WalkArgs::col0) / sizeof(double) >= kMaxNReal, "col0 too small");
  F64Launch L{};
  const bool c0p = B == 1 && h_a != nullptr && p.m >= 1;
  L.fn = tables().f64[cplx ? 1 : 0][c0p ? 1 : 0][p.n];
  PK_REQUIRE(L.fn != nullptr, kErrInternal, "missing fp64 kernel instantiation");
  L.per_warp = B > 1 ? 1 : 0;
  const int elem = cplx ? 16 : 8;
  // minus copies of the columns: F64Walker::kMinus (the C0P kernels)
  const int slot = ((c0p ? 2 : 1) * p.m + 1) * col_stride(p.n, elem) * elem;
  L.smem = slot * (L.per_warp ? kWalkWarps : 1);
  L.occ = occupancy(c, L.fn, kWalkThreads, L.smem);
  const uint64_t units = static_cast<uint64_t>(B) * nt;
  const uint64_t ctas = (units + kWalkWarps - 1) / kWalkWarps;
  L.grid = static_cast<int>(std::min<uint64_t>(ctas, static_cast<uint64_t>(c.sms) * L.occ));
  WalkArgs& a = L.args;
  a.a = d_a;
  a.B = B;
  a.n = p.n;
  a.m = p.m;
  a.algo = algo;
  a.k = p.k;
  a.per_warp_slot = L.per_warp;
  a.tile0 = t0;
  a.tiles = nt;
  a.segs_total = 1ull << (p.m - p.k);
  a.partials = d_partials;
  a.modp_out = nullptr;
  a.primes = nullptr;
  a.want_abs = want_abs ? 1 : 0;
  if (c0p) {  // W[0] as stage_f64 builds it: Ryser a[:, 0], Glynn -2 a[1, :]
    const int n = p.n, w = cplx ? 2 : 1;
    for (int i = 0; i < n; ++i)
      for (int z = 0; z < w; ++z)
        a.col0[w * i + z] = algo == 0 ? h_a[w * (i * n) + z] : -2.0 * h_a[w * (n + i) + z];
#if PK_PAIR4
    std::copy(std::begin(a.col0), std::end(a.col0), std::begin(a.col0b));
#endif
  }
  return L;
}

static void launch_walk(DevCtx& c, const void* fn, int grid, int smem, WalkArgs& args,
                        cudaStream_t st = nullptr) {
  void* kargs[] = {&args};
  PK_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kWalkThreads), kargs, smem, st ? st : c.stream));
}

// Two-stage deterministic reduction of [B][nt] tile partials into [B][5]
// roots; `groups` is scratch of >= B * (nt / group + 2) * 5 doubles.
static void launch_reduce(DevCtx& c, const double* d_partials, int B, uint64_t t0, uint64_t nt,
                          uint64_t group, double* d_groups, double* d_out) {
  const uint64_t g0 = t0 / group, g1 = (t0 + nt - 1) / group + 1;
  const int ng = static_cast<int>(g1 - g0);
  PK_REQUIRE(g1 - g0 <= static_cast<uint64_t>(kMaxGroups) + 1, kErrInternal,
             "too many reduction groups");
  // gridDim.y <= 65535: matrices in slices
  for (int b0 = 0; b0 < B; b0 += 65535) {
    const int nb = std::min(B - b0, 65535);
    dim3 fg((ng + kFoldThreads - 1) / kFoldThreads, nb);
    fold_groups_kernel<<<fg, kFoldThreads, 0, c.stream>>>(
        d_partials + static_cast<size_t>(b0) * nt * kPartialStride, t0, nt, group, g0, ng,
        d_groups + static_cast<size_t>(b0) * ng * kPartialStride);
    PK_CUDA(cudaGetLastError());
  }
  if (d_out == nullptr) return;  // multi-device: the host completes the tree
  tree_groups_kernel<<<B, kTreeThreads, 0, c.stream>>>(d_groups, g0, ng, d_out);
  PK_CUDA(cudaGetLastError());
}

// Host copy of tree_groups_kernel (pk_reduce.cuh): the binary tree over group
// nodes on GLOBAL indices g0 .. g0 + size - 1, a missing child passing its
// sibling through.  With the groups of several devices concatenated in index
// order it reproduces the one-device root bit for bit (pair_combine is
// adds/subtracts only, so there is no contraction to differ).
static Node tree_nodes_host(std::vector<Node> cur, uint64_t g0) {
  uint64_t lo = g0, hi = g0 + cur.size() - 1;
  while (lo != hi) {
    const uint64_t nlo = lo >> 1, nhi = hi >> 1;
    std::vector<Node> nxt;
    nxt.reserve(nhi - nlo + 1);
    for (uint64_t j = nlo; j <= nhi; ++j) {
      const uint64_t l = 2 * j, r = 2 * j + 1;
      const bool hl = l >= lo && l <= hi, hr = r >= lo && r <= hi;
      if (hl && hr)
        nxt.push_back(node_combine_h(cur[l - lo], cur[r - lo]));
      else
        nxt.push_back(hl ? cur[l - lo] : cur[r - lo]);
    }
    cur.swap(nxt);
    lo = nlo;
    hi = nhi;
  }
  return cur[0];
}

static size_t group_scratch_doubles(int B, uint64_t nt, uint64_t group) {
  return static_cast<size_t>(B) * (nt / group + 2) * kPartialStride;
}

// exact-arithmetic pieces on one device; returns one Node per piece.  Piece i
// walks matrix d_a + (i / ppm) * mat_stride (default: every piece, one matrix).
static std::vector<Node> run_f64_pieces(DevCtx& c, const double* d_a, int n, bool cplx, int algo,
                                        const std::vector<std::pair<uint64_t, uint64_t>>& pieces,
                                        bool want_abs, int ppm = 0, size_t mat_stride = 0) {
  std::vector<Node> res(pieces.size());
  if (pieces.empty()) return res;
  const int np = static_cast<int>(pieces.size());
  if (ppm <= 0) ppm = np;
  std::vector<uint64_t> hs(np), hl(np);
  for (int i = 0; i < np; ++i) {
    hs[i] = pieces[i].first;
    hl[i] = pieces[i].second;
  }
  auto* ds = static_cast<uint64_t*>(c.starts.get(np * 8));
  auto* dl = static_cast<uint64_t*>(c.lens.get(np * 8));
  auto* dout = static_cast<double*>(c.blockout.get(np * 4 * 8));
  auto* dabs = static_cast<double*>(c.blockabs.get(np * 8));
  PK_CUDA(cudaMemcpyAsync(ds, hs.data(), np * 8, cudaMemcpyHostToDevice, c.stream));
  PK_CUDA(cudaMemcpyAsync(dl, hl.data(), np * 8, cudaMemcpyHostToDevice, c.stream));
  const int grid = (np + kBlockThreads - 1) / kBlockThreads;
  double* ab = want_abs ? dabs : nullptr;
#define PK_BLOCK(C, A, NM) \
  block_f64_kernel<C, A, NM><<<grid, kBlockThreads, 0, c.stream>>>(d_a, n, ds, dl, np, dout, ab, ppm, mat_stride)
#define PK_BLOCK_N(C, A)                \
  switch (block_nmax(n)) {              \
    case 16: PK_BLOCK(C, A, 16); break; \
    case 32: PK_BLOCK(C, A, 32); break; \
    case 48: PK_BLOCK(C, A, 48); break; \
    default: PK_BLOCK(C, A, 64); break; \
  }
  if (cplx) {
    if (algo == 0)
      PK_BLOCK_N(true, 0)
    else
      PK_BLOCK_N(true, 1)
  } else {
    if (algo == 0)
      PK_BLOCK_N(false, 0)
    else
      PK_BLOCK_N(false, 1)
  }
#undef PK_BLOCK_N
#undef PK_BLOCK
  PK_CUDA(cudaGetLastError());
  std::vector<double> h(np * 4), habs(np, 0.0);
  PK_CUDA(cudaMemcpyAsync(h.data(), dout, np * 4 * 8, cudaMemcpyDeviceToHost, c.stream));
  if (want_abs)
    PK_CUDA(cudaMemcpyAsync(habs.data(), dabs, np * 8, cudaMemcpyDeviceToHost, c.stream));
  PK_CUDA(cudaStreamSynchronize(c.stream));
  for (int i = 0; i < np; ++i)
    res[i] = Node{Pair{h[4 * i], h[4 * i + 2]}, Pair{h[4 * i + 1], h[4 * i + 3]}, habs[i]};
  return res;
}

// Run `fn(dev_index)` on devices [0, ndev) with one host thread per device.
template <class F>
static void for_devices(int ndev, F&& fn) {
  if (ndev <= 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::string> err(ndev);
  std::vector<int> code(ndev, 0);
  for (int d = 0; d < ndev; ++d) {
    th.emplace_back([&, d] {
      try {
        fn(d);
      } catch (const Error& e) {
        err[d] = e.what();
        code[d] = e.code;
      } catch (const std::exception& e) {
        err[d] = e.what();
        code[d] = kErrInternal;
      }
    });
  }
  for (auto& t : th) t.join();
  for (int d = 0; d < ndev; ++d)
    if (code[d]) fail(code[d], "device " + std::to_string(d) + ": " + err[d]);
}

static int clamp_ndev(int ndev) {
  const int nd = device_count() - g_device_base.load();
  PK_REQUIRE(nd > 0, kErrCuda, "no CUDA device visible");
  return std::max(1, std::min(ndev, nd));
}

static void check_f64_args(const double* a, int n, int algo) {
  PK_REQUIRE(a != nullptr, kErrArg, "null matrix pointer");
  PK_REQUIRE(n >= 1, kErrArg, "empty matrix");
  PK_REQUIRE(algo == 0 || algo == 1, kErrArg, "algo must be 0 (ryser) or 1 (glynn)");
  PK_REQUIRE(n <= kBlockMaxN, kErrLimit, "dimension exceeds 64");
}

static void check_range(int m, uint64_t start, uint64_t length) {
  const uint64_t total = m >= 64 ? ~0ull : (1ull << m);
  PK_REQUIRE(start <= total && length <= total - start, kErrArg,
             "Gray range [start, start+length) exceeds 2^m");
}

// ---------------------------------------------------------------------------
// F_p host arithmetic

using u128 = unsigned __int128;
static uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t p) {
  return static_cast<uint64_t>(static_cast<u128>(a) * b % p);
}
static uint64_t powmod_h(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  b %= p;
  while (e) {
    if (e & 1) r = mulmod_h(r, b, p);
    b = mulmod_h(b, b, p);
    e >>= 1;
  }
  return r;
}
// 2^(bits * reps) mod p
static uint64_t pow2mod_h(uint64_t bits_times_reps, uint64_t p) { return powmod_h(2, bits_times_reps, p); }

static bool fast_prime(uint64_t p) { return (p & 1) && p >= 3 && p < (1ull << 31); }
// odd moduli for the Montgomery-64 walk (pk_walk64.cuh)
static bool wide_prime(uint64_t p) { return (p & 1) && p >= (1ull << 31) && p < (1ull << 62); }
// either register-resident F_p walk
static bool walk_prime(uint64_t p) { return fast_prime(p) || wide_prime(p); }
// exact integer row sums fit 31 bits: n (p - 1) < 2^31
static bool lazy_prime(uint64_t p, int n) {
  return fast_prime(p) && static_cast<uint64_t>(n) * (p - 1) < (1ull << 31);
}

}  // namespace pk

// ===========================================================================
// extern "C"

using namespace pk;

extern "C" const char* pk_last_error(void) { return last_error_cstr(); }

extern "C" int pk_version(void) { return 100; }

extern "C" int pk_max_n(void) { return kMaxN; }

extern "C" int pk_device_count(void) {
  return pk_guard([&]() -> int { return device_count(); });
}

extern "C" int pk_set_logical_devices(int count) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(count >= 0 && count <= 64, kErrArg, "logical device count must be in [0, 64]");
    g_logical.store(count);
    return 0;
  });
}

extern "C" int pk_set_device_base(int base) {
  return pk_guard([&]() -> int {
    const int nd = device_count();
    PK_REQUIRE(base >= 0 && (base < nd || (nd == 0 && base == 0)), kErrArg,
               "device base " + std::to_string(base) + " outside the " + std::to_string(nd) +
                   " visible devices");
    g_device_base.store(base);
    return 0;
  });
}

namespace pk {

// fp64 range on ndev devices.
//
// One device: walk + fold + tree on the device, one root.  Several devices: the
// aligned tile interior is cut at reduction-group boundaries, each device walks
// its share and folds its groups, and the host runs the group tree over all
// devices' groups in global order (tree_nodes_host) -- bit-identical to one
// device for ANY cut, aligned or not.  The ragged head / tail pieces (exact
// kernel) are dealt round-robin over the devices and folded in index order.
static Node f64_range(const double* a, int n, bool cplx, int algo, uint64_t start,
                      uint64_t length, int ndev, bool want_abs) {
  check_f64_args(a, n, algo);
  const Plan p = make_plan(n, algo);
  check_range(p.m, start, length);
  const Range r = make_range(p, start, length);
  const size_t abytes = static_cast<size_t>(n) * n * (cplx ? 16 : 8);
  const uint64_t nt = r.t1 - r.t0;
  std::vector<std::pair<uint64_t, uint64_t>> pcs = r.head;
  pcs.insert(pcs.end(), r.tail.begin(), r.tail.end());
  ndev = (nt || pcs.size() > 1) ? clamp_ndev(ndev) : 1;
  // interior cut on group boundaries (groups never straddle devices)
  std::vector<uint64_t> cut(ndev + 1);
  for (int d = 0; d <= ndev; ++d) {
    uint64_t t = r.t0 + nt * d / ndev;
    if (d > 0 && d < ndev) t = std::max(r.t0, std::min(r.t1, (t + p.group / 2) / p.group * p.group));
    cut[d] = t;
  }
  Node root{};
  std::vector<std::vector<Node>> dev_groups(ndev);
  std::vector<uint64_t> dev_g0(ndev, 0);
  std::vector<Node> pres(pcs.size());
  for_devices(ndev, [&](int d) {
    DevCtx& c = ctx(d);
    std::lock_guard<std::mutex> g(c.mu);
    PK_CUDA(cudaSetDevice(c.dev));
    auto* d_a = static_cast<double*>(c.a.get(abytes));
    PK_CUDA(cudaMemcpyAsync(d_a, a, abytes, cudaMemcpyHostToDevice, c.stream));
    const uint64_t t0 = cut[d], t1 = cut[d + 1];
    if (t1 > t0) {
      auto* d_part = static_cast<double*>(c.partials.get((t1 - t0) * kPartialStride * 8));
      F64Launch L = prepare_f64(c, p, cplx, algo, 1, d_a, t0, t1 - t0, want_abs, d_part, a);
      launch_walk(c, L.fn, L.grid, L.smem, L.args);
      auto* d_grp = static_cast<double*>(c.groups.get(group_scratch_doubles(1, t1 - t0, p.group) * 8));
      if (ndev == 1) {
        auto* d_out = static_cast<double*>(c.out.get(kPartialStride * 8));
        launch_reduce(c, d_part, 1, t0, t1 - t0, p.group, d_grp, d_out);
        double h[kPartialStride];
        PK_CUDA(cudaMemcpyAsync(h, d_out, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        PK_CUDA(cudaStreamSynchronize(c.stream));
        root = node_from5(h);
      } else {
        launch_reduce(c, d_part, 1, t0, t1 - t0, p.group, d_grp, nullptr);
        const uint64_t g0 = t0 / p.group, g1 = (t1 - 1) / p.group + 1;
        std::vector<double> h((g1 - g0) * kPartialStride);
        PK_CUDA(cudaMemcpyAsync(h.data(), d_grp, h.size() * 8, cudaMemcpyDeviceToHost, c.stream));
        PK_CUDA(cudaStreamSynchronize(c.stream));
        dev_g0[d] = g0;
        for (uint64_t gi = 0; gi < g1 - g0; ++gi) dev_groups[d].push_back(node_from5(&h[gi * kPartialStride]));
      }
    }
    std::vector<std::pair<uint64_t, uint64_t>> mine;
    for (size_t i = d; i < pcs.size(); i += ndev) mine.push_back(pcs[i]);
    const std::vector<Node> v = run_f64_pieces(c, d_a, n, cplx, algo, mine, want_abs);
    for (size_t i = d, j = 0; i < pcs.size(); i += ndev, ++j) pres[i] = v[j];
  });
  if (ndev > 1 && nt) {
    std::vector<Node> all;
    uint64_t g0 = 0;
    bool first = true;
    for (int d = 0; d < ndev; ++d) {
      if (dev_groups[d].empty()) continue;
      if (first) g0 = dev_g0[d];
      first = false;
      all.insert(all.end(), dev_groups[d].begin(), dev_groups[d].end());
    }
    root = tree_nodes_host(std::move(all), g0);
  }
  // index order: head pieces, the interior root, tail pieces
  std::vector<Node> seq(pres.begin(), pres.begin() + r.head.size());
  if (nt) seq.push_back(root);
  seq.insert(seq.end(), pres.begin() + r.head.size(), pres.end());
  if (seq.empty()) return Node{};
  Node acc = seq[0];
  for (size_t i = 1; i < seq.size(); ++i) acc = node_combine_h(acc, seq[i]);
  return acc;
}

}  // namespace pk

extern "C" int pk_ryser_f64(const double* a, int n, int is_complex, int algo, uint64_t start,
                            uint64_t length, int ndev, double out[4], double* abs_sum) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(out != nullptr, kErrArg, "null output pointer");
    const Node v = f64_range(a, n, is_complex != 0, algo, start, length, ndev, abs_sum != nullptr);
    out[0] = v.re.s;
    out[1] = v.im.s;
    out[2] = v.re.c;
    out[3] = v.im.c;
    if (abs_sum) *abs_sum = v.ab;
    return 0;
  });
}

namespace pk {

// A caller's block plan on one device: blocks [b0, b1).  Every block gets the
// root and pieces a single-range call on it would (same plan, groups, tree and
// piece cuts), so node[b] is bit-identical to f64_range on the block.  The
// aligned interiors are walked in as few launches as possible (runs of blocks
// whose interiors are adjacent up to a few tiles share one launch), then one
// segmented fold and one segmented tree reduce every block, and one exact
// launch walks every block's ragged pieces.
static void f64_plan_device(DevCtx& c, const double* a, int n, bool cplx, int algo, const Plan& p,
                            const std::vector<Range>& rs, int b0, int b1, bool want_abs,
                            std::vector<Node>& node) {
  const size_t abytes = static_cast<size_t>(n) * n * (cplx ? 16 : 8);
  auto* d_a = static_cast<double*>(c.a.get(abytes));
  PK_CUDA(cudaMemcpyAsync(d_a, a, abytes, cudaMemcpyHostToDevice, c.stream));
  // runs of interiors (blocks in order; a gap of <= 4 tiles is walked, not split)
  struct Run {
    uint64_t lo, hi, pidx;
  };
  std::vector<Run> runs;
  std::vector<uint64_t> pbase(b1 - b0, 0);
  uint64_t ptotal = 0;
  for (int b = b0; b < b1; ++b) {
    const Range& r = rs[b];
    if (r.t1 <= r.t0) continue;
    if (!runs.empty() && r.t0 >= runs.back().lo && r.t0 <= runs.back().hi + 4) {
      Run& u = runs.back();
      if (r.t1 > u.hi) {
        ptotal += r.t1 - u.hi;
        u.hi = r.t1;
      }
    } else {
      runs.push_back(Run{r.t0, r.t1, ptotal});
      ptotal += r.t1 - r.t0;
    }
    const Run& u = runs.back();
    pbase[b - b0] = u.pidx + (r.t0 - u.lo);
  }
  std::vector<FoldTask> ft;
  std::vector<TreeTask> tt;
  std::vector<int> tree_block;
  for (int b = b0; b < b1; ++b) {
    const Range& r = rs[b];
    if (r.t1 <= r.t0) continue;
    const uint64_t g0 = r.t0 / p.group, g1 = (r.t1 - 1) / p.group + 1;
    tt.push_back(TreeTask{g0, static_cast<int>(ft.size()), static_cast<int>(g1 - g0)});
    tree_block.push_back(b);
    for (uint64_t g = g0; g < g1; ++g) {
      const uint64_t lo = std::max(g * p.group, r.t0), hi = std::min((g + 1) * p.group, r.t1);
      ft.push_back(FoldTask{lo, hi, pbase[b - b0] + (lo - r.t0)});
    }
  }
  if (!runs.empty()) {
    auto* d_part = static_cast<double*>(c.partials.get(ptotal * kPartialStride * 8));
    for (const Run& u : runs) {
      F64Launch L = prepare_f64(c, p, cplx, algo, 1, d_a, u.lo, u.hi - u.lo, want_abs,
                                d_part + u.pidx * kPartialStride, a);
      launch_walk(c, L.fn, L.grid, L.smem, L.args);
    }
    // task tables and group nodes share the `groups` scratch: tasks first
    const size_t ft_bytes = (ft.size() * sizeof(FoldTask) + 255) & ~size_t(255);
    const size_t tt_bytes = (tt.size() * sizeof(TreeTask) + 255) & ~size_t(255);
    auto* scratch = static_cast<uint8_t*>(
        c.groups.get(ft_bytes + tt_bytes + ft.size() * kPartialStride * 8));
    auto* d_ft = reinterpret_cast<FoldTask*>(scratch);
    auto* d_tt = reinterpret_cast<TreeTask*>(scratch + ft_bytes);
    auto* d_grp = reinterpret_cast<double*>(scratch + ft_bytes + tt_bytes);
    auto* d_out = static_cast<double*>(c.out.get(tt.size() * kPartialStride * 8));
    PK_CUDA(cudaMemcpyAsync(d_ft, ft.data(), ft.size() * sizeof(FoldTask), cudaMemcpyHostToDevice,
                            c.stream));
    PK_CUDA(cudaMemcpyAsync(d_tt, tt.data(), tt.size() * sizeof(TreeTask), cudaMemcpyHostToDevice,
                            c.stream));
    const int nft = static_cast<int>(ft.size());
    fold_tasks_kernel<<<(nft + kFoldThreads - 1) / kFoldThreads, kFoldThreads, 0, c.stream>>>(
        d_part, d_ft, nft, d_grp);
    PK_CUDA(cudaGetLastError());
    tree_tasks_kernel<<<static_cast<int>(tt.size()), kTreeThreads, 0, c.stream>>>(d_grp, d_tt, d_out);
    PK_CUDA(cudaGetLastError());
    std::vector<double> h(tt.size() * kPartialStride);
    PK_CUDA(cudaMemcpyAsync(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost, c.stream));
    PK_CUDA(cudaStreamSynchronize(c.stream));
    for (size_t i = 0; i < tt.size(); ++i) node[tree_block[i]] = node_from5(&h[i * kPartialStride]);
  }
  // every block's ragged pieces in one exact launch, then the index-order fold
  std::vector<std::pair<uint64_t, uint64_t>> pcs;
  for (int b = b0; b < b1; ++b) {
    pcs.insert(pcs.end(), rs[b].head.begin(), rs[b].head.end());
    pcs.insert(pcs.end(), rs[b].tail.begin(), rs[b].tail.end());
  }
  const std::vector<Node> pv = run_f64_pieces(c, d_a, n, cplx, algo, pcs, want_abs);
  size_t k = 0;
  for (int b = b0; b < b1; ++b) {
    const Range& r = rs[b];
    std::vector<Node> seq(pv.begin() + k, pv.begin() + k + r.head.size());
    k += r.head.size();
    if (r.t1 > r.t0) seq.push_back(node[b]);
    seq.insert(seq.end(), pv.begin() + k, pv.begin() + k + r.tail.size());
    k += r.tail.size();
    Node acc{};
    if (!seq.empty()) {
      acc = seq[0];
      for (size_t i = 1; i < seq.size(); ++i) acc = node_combine_h(acc, seq[i]);
    }
    node[b] = acc;
  }
}

}  // namespace pk

extern "C" int pk_ryser_f64_plan(const double* a, int n, int is_complex, int algo,
                                 const uint64_t* starts, const uint64_t* lens, int nblocks,
                                 int ndev, double* out, double* abs_sums) {
  return pk_guard([&]() -> int {
    check_f64_args(a, n, algo);
    PK_REQUIRE(nblocks >= 0, kErrArg, "negative block count");
    if (nblocks == 0) return 0;
    PK_REQUIRE(starts && lens && out, kErrArg, "null block arrays");
    const bool cplx = is_complex != 0;
    const Plan p = make_plan(n, algo);
    std::vector<Range> rs(nblocks);
    for (int b = 0; b < nblocks; ++b) {
      check_range(p.m, starts[b], lens[b]);
      rs[b] = make_range(p, starts[b], lens[b]);
    }
    ndev = std::min(clamp_ndev(ndev), nblocks);
    std::vector<Node> node(nblocks);
    for_devices(ndev, [&](int d) {
      const int b0 = static_cast<int>(static_cast<int64_t>(nblocks) * d / ndev);
      const int b1 = static_cast<int>(static_cast<int64_t>(nblocks) * (d + 1) / ndev);
      if (b1 <= b0) return;
      DevCtx& c = ctx(d);
      std::lock_guard<std::mutex> g(c.mu);
      PK_CUDA(cudaSetDevice(c.dev));
      f64_plan_device(c, a, n, cplx, algo, p, rs, b0, b1, abs_sums != nullptr, node);
    });
    for (int b = 0; b < nblocks; ++b) {
      out[4 * b + 0] = node[b].re.s;
      out[4 * b + 1] = node[b].im.s;
      out[4 * b + 2] = node[b].re.c;
      out[4 * b + 3] = node[b].im.c;
      if (abs_sums) abs_sums[b] = node[b].ab;
    }
    return 0;
  });
}

// The reference's ordered combine of block partials (engine.py:240-245:
// KahanAccumulator add(s); add(c) per block, Neumaier per component,
// engine.py:33-73), so that a plan of thousands of blocks costs no Python loop.
extern "C" int pk_kahan_fold(const double* pairs, int nblocks, int is_complex, double out[4]) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(nblocks >= 0 && (nblocks == 0 || pairs) && out, kErrArg, "bad fold arguments");
    double s[2] = {0.0, 0.0}, c[2] = {0.0, 0.0};
    auto add = [&](int z, double v) {
      const double t = s[z] + v;
      const bool big_s = std::fabs(s[z]) >= std::fabs(v);
      c[z] += big_s ? ((s[z] - t) + v) : ((v - t) + s[z]);
      s[z] = t;
    };
    for (int b = 0; b < nblocks; ++b) {
      const double* q = pairs + 4 * b;  // s_re, s_im, c_re, c_im
      add(0, q[0]);
      if (is_complex) add(1, q[1]);
      add(0, q[2]);
      if (is_complex) add(1, q[3]);
    }
    out[0] = s[0];
    out[1] = s[1];
    out[2] = c[0];
    out[3] = c[1];
    return 0;
  });
}

extern "C" int pk_ryser_f64_blocks(const double* a, int n, int is_complex, int algo,
                                   const uint64_t* starts, const uint64_t* lens, int nblocks,
                                   int device, double* out) {
  return pk_guard([&]() -> int {
    check_f64_args(a, n, algo);
    PK_REQUIRE(nblocks >= 0, kErrArg, "negative block count");
    if (nblocks == 0) return 0;
    PK_REQUIRE(starts && lens && out, kErrArg, "null block arrays");
    const int m = algo == 0 ? n : n - 1;
    for (int i = 0; i < nblocks; ++i) check_range(m, starts[i], lens[i]);
    DevCtx& c = ctx(device);
    std::lock_guard<std::mutex> g(c.mu);
    PK_CUDA(cudaSetDevice(c.dev));
    const size_t abytes = static_cast<size_t>(n) * n * (is_complex ? 16 : 8);
    auto* d_a = static_cast<double*>(c.a.get(abytes));
    PK_CUDA(cudaMemcpyAsync(d_a, a, abytes, cudaMemcpyHostToDevice, c.stream));
    std::vector<std::pair<uint64_t, uint64_t>> pcs(nblocks);
    for (int i = 0; i < nblocks; ++i) pcs[i] = {starts[i], lens[i]};
    const std::vector<Node> v = run_f64_pieces(c, d_a, n, is_complex != 0, algo, pcs, false);
    for (int i = 0; i < nblocks; ++i) {
      out[4 * i + 0] = v[i].re.s;
      out[4 * i + 1] = v[i].im.s;
      out[4 * i + 2] = v[i].re.c;
      out[4 * i + 3] = v[i].im.c;
    }
    return 0;
  });
}

extern "C" int pk_ryser_f64_batch(const double* a, int B, int n, int is_complex, int algo,
                                  int ndev, double* out, double* abs_sums) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(B >= 0, kErrArg, "negative batch size");
    if (B == 0) return 0;
    check_f64_args(a, n, algo);
    PK_REQUIRE(out != nullptr, kErrArg, "null output pointer");
    const bool cplx = is_complex != 0;
    const size_t mat = static_cast<size_t>(n) * n * (cplx ? 2 : 1);
    ndev = clamp_ndev(ndev);
    ndev = std::min(ndev, B);
    for_devices(ndev, [&](int d) {
      const int b0 = static_cast<int>(static_cast<int64_t>(B) * d / ndev);
      const int b1 = static_cast<int>(static_cast<int64_t>(B) * (d + 1) / ndev);
      const int nb = b1 - b0;
      if (nb <= 0) return;
      DevCtx& c = ctx(d);
      std::lock_guard<std::mutex> g(c.mu);
      PK_CUDA(cudaSetDevice(c.dev));
      const Plan p = make_plan(n, algo);
      auto* d_a = static_cast<double*>(c.a.get(nb * mat * 8));
      PK_CUDA(cudaMemcpyAsync(d_a, a + b0 * mat, nb * mat * 8, cudaMemcpyHostToDevice, c.stream));
      std::vector<double> h(static_cast<size_t>(nb) * kPartialStride);
      if (p.k > 0 && batch_per_matrix(p.m, cplx)) {
        // one C0P launch per matrix over the aux streams; sub-batches bound the
        // partials buffer; one reduce per sub-batch on the main stream
        const Plan p1 = make_plan_per_matrix(n, algo);
        const uint64_t nt = p1.tiles_total;
        c.ensure_aux();
        const int sb = subbatch_cap(
            static_cast<int>(std::clamp<uint64_t>((1ull << 24) / (nt * kPartialStride), 1, nb)));
        auto* d_part = static_cast<double*>(c.partials.get(sb * nt * kPartialStride * 8));
        auto* d_out = static_cast<double*>(c.out.get(nb * kPartialStride * 8));
        auto* d_grp = static_cast<double*>(c.groups.get(group_scratch_doubles(sb, nt, p1.group) * 8));
        for (int s0 = 0; s0 < nb; s0 += sb) {
          const int ns = std::min(sb, nb - s0);
          PK_CUDA(cudaEventRecord(c.ev_main, c.stream));  // input copied, previous reduce done
          const int nst = batch_streams();
          for (int i = 0; i < nst; ++i) PK_CUDA(cudaStreamWaitEvent(c.aux[i], c.ev_main, 0));
          for (int b = 0; b < ns; ++b) {
            const size_t off = static_cast<size_t>(s0 + b) * mat;
            F64Launch L = prepare_f64(c, p1, cplx, algo, 1, d_a + off, 0, nt, abs_sums != nullptr,
                                      d_part + b * nt * kPartialStride, a + b0 * mat + off);
            launch_walk(c, L.fn, L.grid, L.smem, L.args, c.aux[b % nst]);
          }
          for (int i = 0; i < nst; ++i) {
            PK_CUDA(cudaEventRecord(c.ev_aux[i], c.aux[i]));
            PK_CUDA(cudaStreamWaitEvent(c.stream, c.ev_aux[i], 0));
          }
          launch_reduce(c, d_part, ns, 0, nt, p1.group, d_grp, d_out + s0 * kPartialStride);
        }
        PK_CUDA(cudaMemcpyAsync(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost, c.stream));
        PK_CUDA(cudaStreamSynchronize(c.stream));
      } else if (p.k > 0) {
        // a matrix per warp slot; sub-batches of <= 2^17 tiles bound the partials
        const uint64_t nt = p.tiles_total;
        const int sb = subbatch_cap(static_cast<int>(std::clamp<uint64_t>((1ull << 17) / nt, 1, nb)));
        auto* d_part = static_cast<double*>(c.partials.get(sb * nt * kPartialStride * 8));
        auto* d_out = static_cast<double*>(c.out.get(nb * kPartialStride * 8));
        auto* d_grp = static_cast<double*>(c.groups.get(group_scratch_doubles(sb, nt, p.group) * 8));
        for (int s0 = 0; s0 < nb; s0 += sb) {
          const int ns = std::min(sb, nb - s0);
          const size_t off = static_cast<size_t>(s0) * mat;
          F64Launch L = prepare_f64(c, p, cplx, algo, ns, d_a + off, 0, nt, abs_sums != nullptr,
                                    d_part, a + b0 * mat + off);
          launch_walk(c, L.fn, L.grid, L.smem, L.args);
          launch_reduce(c, d_part, ns, 0, nt, p.group, d_grp, d_out + s0 * kPartialStride);
        }
        PK_CUDA(cudaMemcpyAsync(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost, c.stream));
        PK_CUDA(cudaStreamSynchronize(c.stream));
      } else {
        // tiny m: one exact piece per matrix (2^m <= 32 terms), all in one launch
        std::vector<std::pair<uint64_t, uint64_t>> pcs(nb, {0, 1ull << p.m});
        const std::vector<Node> v =
            run_f64_pieces(c, d_a, n, cplx, algo, pcs, abs_sums != nullptr, 1, mat);
        for (int b = 0; b < nb; ++b) {
          const Node& x = v[b];
          double* o = h.data() + b * kPartialStride;
          o[0] = x.re.s;
          o[1] = x.re.c;
          o[2] = x.im.s;
          o[3] = x.im.c;
          o[4] = x.ab;
        }
      }
      for (int b = 0; b < nb; ++b) {
        const double* o = h.data() + b * kPartialStride;
        double* r = out + 4 * static_cast<size_t>(b0 + b);
        r[0] = o[0];
        r[1] = o[2];
        r[2] = o[1];
        r[3] = o[3];
        if (abs_sums) abs_sums[b0 + b] = o[4];
      }
    });
    return 0;
  });
}

// ---------------------------------------------------------------------------
// F_p

namespace pk {

struct ModpGroup {
  int P;                       // primes in the launch group (<= kMaxP)
  bool lazy;                   // unreduced row sums (n p < 2^31) or reduced [0, p)
  int pf = 0;                  // trailing fp64 primes (hybrid kernel, lazy only)
  std::vector<int> idx;        // indices into the caller's prime list
  bool wide = false;           // Montgomery-64 walk: 64-bit residues, 2 output words per prime
  bool wf = false;             // hybrid with a wide fp64 prime (fp64w_prime_ok, two-product)
  int out_words() const { return wide ? 2 * P : P; }
};

// raw -> exact residue of the fast kernel: raw * sgn0 * 2^(32 (n-1)) mod p
static uint64_t fix_fast(uint64_t raw, uint64_t p, int n, int algo) {
  uint64_t v = mulmod_h(raw % p, pow2mod_h(32ull * (n - 1), p), p);
  if (algo == 0 && (n & 1)) v = v == 0 ? 0 : p - v;
  return v;
}
// raw -> exact residue of an fp64 (hybrid) prime: plain sum, Ryser sign only
static uint64_t fix_fp64(uint64_t raw, uint64_t p, int n, int algo) {
  uint64_t v = raw % p;
  if (algo == 0 && (n & 1)) v = v == 0 ? 0 : p - v;
  return v;
}
// (lo, hi) 128-bit counter of the wide walk -> residue: * 2^(64 n), Ryser sign
static uint64_t fix_wide(uint64_t lo, uint64_t hi, uint64_t p, int n, int algo) {
  const uint64_t raw = static_cast<uint64_t>(((static_cast<u128>(hi) << 64) | lo) % p);
  uint64_t v = mulmod_h(raw, pow2mod_h(64ull * n, p), p);
  if (algo == 0 && (n & 1)) v = v == 0 ? 0 : p - v;
  return v;
}
static uint64_t fix_block(uint64_t raw, uint64_t p, int n) {
  if (!(p & 1)) return raw % p;
  return mulmod_h(raw % p, pow2mod_h(64ull * (n - 1), p), p);
}
// the group's residue matrices as the kernel reads them: uint32 for the
// Montgomery-32 primes, uint64 for the wide walk and for the fp64 primes of a
// hybrid group (after the uint32 part, padded to 8 bytes: hybrid_fp_offset)
static std::vector<uint8_t> pack_residues(const ModpGroup& G, const uint64_t* a, size_t nn) {
  std::vector<uint8_t> h;
  const int pi = G.P - G.pf;
  for (int q = 0; q < G.P; ++q) {
    const bool w64 = G.wide || q >= pi;
    if (w64 && (h.size() & 7)) h.resize((h.size() + 7) & ~size_t(7), 0);
    const uint64_t* aq = a + G.idx[q] * nn;
    for (size_t e = 0; e < nn; ++e) {
      const size_t o = h.size();
      if (w64) {
        h.resize(o + 8);
        std::memcpy(&h[o], &aq[e], 8);
      } else {
        const uint32_t v = static_cast<uint32_t>(aq[e]);
        h.resize(o + 4);
        std::memcpy(&h[o], &v, 4);
      }
    }
  }
  if (h.size() & 7) h.resize((h.size() + 7) & ~size_t(7), 0);  // next group stays aligned
  return h;
}
// one launch group's raw output words -> residues, stored at the caller's indices
static void decode_group(const ModpGroup& G, const unsigned long long* ho, const uint64_t* primes,
                         int n, int algo, uint64_t* res) {
  for (int q = 0; q < G.P; ++q) {
    const int k = G.idx[q];
    if (G.wide)
      res[k] = fix_wide(ho[2 * q], ho[2 * q + 1], primes[k], n, algo);
    else if (q >= G.P - G.pf)
      res[k] = fix_fp64(ho[q], primes[k], n, algo);
    else
      res[k] = fix_fast(ho[q], primes[k], n, algo);
  }
}

// generic walker for one modulus over pieces; returns the residue sum
static uint64_t modp_pieces(DevCtx& c, const uint64_t* d_a, int n, int algo, uint64_t p,
                            const std::vector<std::pair<uint64_t, uint64_t>>& pieces) {
  if (pieces.empty()) return 0;
  const int np = static_cast<int>(pieces.size());
  std::vector<uint64_t> hs(np), hl(np), ho(np);
  for (int i = 0; i < np; ++i) {
    hs[i] = pieces[i].first;
    hl[i] = pieces[i].second;
  }
  auto* ds = static_cast<uint64_t*>(c.starts.get(np * 8));
  auto* dl = static_cast<uint64_t*>(c.lens.get(np * 8));
  auto* dout = static_cast<uint64_t*>(c.blockout.get(np * 8));
  PK_CUDA(cudaMemcpyAsync(ds, hs.data(), np * 8, cudaMemcpyHostToDevice, c.stream));
  PK_CUDA(cudaMemcpyAsync(dl, hl.data(), np * 8, cudaMemcpyHostToDevice, c.stream));
  const int grid = (np + kBlockThreads - 1) / kBlockThreads;
#define PK_BLOCKP(A, NM) block_modp_kernel<A, NM><<<grid, kBlockThreads, 0, c.stream>>>(d_a, n, p, ds, dl, np, dout)
#define PK_BLOCKP_N(A)                \
  switch (block_nmax(n)) {            \
    case 16: PK_BLOCKP(A, 16); break; \
    case 32: PK_BLOCKP(A, 32); break; \
    case 48: PK_BLOCKP(A, 48); break; \
    default: PK_BLOCKP(A, 64); break; \
  }
  if (algo == 0)
    PK_BLOCKP_N(0)
  else
    PK_BLOCKP_N(1)
#undef PK_BLOCKP_N
#undef PK_BLOCKP
  PK_CUDA(cudaGetLastError());
  PK_CUDA(cudaMemcpyAsync(ho.data(), dout, np * 8, cudaMemcpyDeviceToHost, c.stream));
  PK_CUDA(cudaStreamSynchronize(c.stream));
  uint64_t s = 0;
  for (int i = 0; i < np; ++i) s = static_cast<uint64_t>((static_cast<u128>(s) + ho[i]) % p);
  return fix_block(s, p, n);
}

struct ModpLaunch {
  const void* fn;
  int grid, smem, occ;
  WalkArgs args;
};

// One launch per prime group: constants go into the kernel's grid-constant
// parameter (args.mc); `group_primes` lists the group's moduli (the last `pf`
// of them are fp64 primes of the hybrid kernel).
static ModpLaunch prepare_modp(DevCtx& c, const Plan& p, const ModpGroup& G, int algo,
                               const void* d_a, const std::vector<uint64_t>& group_primes,
                               uint64_t t0, uint64_t nt, unsigned long long* d_out) {
  const bool lazy = G.lazy;
  const int pf = G.pf;
  PK_REQUIRE(p.n >= 1 && p.n <= kMaxN, kErrLimit,
             "dimension " + std::to_string(p.n) + " exceeds the GPU kernel range n <= " +
                 std::to_string(kMaxN));
  const int P = static_cast<int>(group_primes.size());
  const int pi = P - pf;
  ModpLaunch L{};
  if (G.wide) {
    PK_REQUIRE(P >= 1 && P <= kMaxPWide, kErrInternal, "bad wide prime group");
    bool lazy64 = true;  // rows reduced every second step needs p < 2^60 (pk_walk64.cuh)
    for (int q = 0; q < P; ++q) lazy64 = lazy64 && group_primes[q] < (1ull << 60);
    L.fn = tables().wide[lazy64 ? 1 : 0][P][p.n];
    PK_REQUIRE(L.fn != nullptr, kErrInternal, "missing wide F_p kernel instantiation");
    L.smem = (2 * p.m + 1) * P * col_stride(p.n, 8) * 8;
  } else if (pf) {
    PK_REQUIRE(pi == 1 && pf == 1, kErrInternal, "hybrid groups are one lazy + one fp64 prime");
    L.fn = tables().hybrid[G.wf ? 1 : 0][p.n];
    PK_REQUIRE(L.fn != nullptr, kErrInternal, "missing hybrid F_p kernel instantiation");
    const int int_words = ((2 * p.m + 1) * pi * col_stride(p.n, 4) + 1) & ~1;
    L.smem = int_words * 4 + (2 * p.m + 1) * pf * col_stride(p.n, 8) * 8;
  } else {
    L.fn = tables().modp[lazy ? 1 : 0][P][p.n];
    PK_REQUIRE(L.fn != nullptr, kErrInternal, "missing F_p kernel instantiation");
    L.smem = (2 * p.m + 1) * P * col_stride(p.n, 4) * 4;
  }
  L.occ = occupancy(c, L.fn, kWalkThreads, L.smem);
  const uint64_t ctas = (nt + kWalkWarps - 1) / kWalkWarps;
  L.grid = static_cast<int>(std::min<uint64_t>(ctas, static_cast<uint64_t>(c.sms) * L.occ));
  WalkArgs& a = L.args;
  a.a = d_a;
  a.B = 1;
  a.n = p.n;
  a.m = p.m;
  a.algo = algo;
  a.k = p.k;
  a.per_warp_slot = 0;
  a.tile0 = t0;
  a.tiles = nt;
  a.segs_total = 1ull << (p.m - p.k);
  a.partials = nullptr;
  a.modp_out = d_out;
  a.primes = nullptr;
  a.want_abs = 0;
  for (int q = 0; G.wide && q < P; ++q) {
    a.mc.p64[q] = group_primes[q];
    a.mc.pinv64[q] = 0ull - mont_neg_inv64(group_primes[q]);
  }
  for (int q = 0; !G.wide && q < pi; ++q) {
    const uint32_t pq = static_cast<uint32_t>(group_primes[q]);
    a.mc.p[q] = pq;
    a.mc.mneg[q] = mont_neg_inv32(pq);
    // REDC outputs stay below 2p (reduced rows) or 2^30 + p (lazy rows)
    a.mc.kneg[q] = lazy ? pq * ((1u << 30) / pq + 2u) : 2u * pq;
  }
  for (int q = 0; q < pf; ++q) {
    a.mc.fp[q] = static_cast<double>(group_primes[pi + q]);
    a.mc.fpinv[q] = 1.0 / a.mc.fp[q];
  }
  return L;
}

// Primes per lane: four while the register-resident state (P x n words) fits
// without spilling, three for n > 36.
static int max_primes_per_lane(int n) { return n <= 36 ? kMaxP : 3; }

static bool hybrid_available(int n) { return n >= kHybridMinN && n <= kMaxN; }

// Launch groups: each fp64-eligible prime is paired with one Montgomery prime
// in a hybrid (1 + 1) group while both kinds remain; the rest go in groups of
// up to max_primes_per_lane(n) primes of one row mode.
static std::vector<ModpGroup> group_primes(const std::vector<int>& fast, const uint64_t* primes,
                                           int n) {
  std::vector<ModpGroup> gs;
  const int pmax = max_primes_per_lane(n);
  std::vector<int> fp, fpw, lz, red, wd;
  for (int k : fast) {
    if (wide_prime(primes[k]) && fp64w_prime_ok(primes[k], n) && hybrid_available(n))
      fpw.push_back(k);  // pairs with a lazy prime below, else the Montgomery-64 walk
    else if (wide_prime(primes[k]))
      wd.push_back(k);
    else if (!lazy_prime(primes[k], n))
      red.push_back(k);
    else if (fp64_prime_ok(primes[k], n))
      fp.push_back(k);
    else
      lz.push_back(k);
  }
  if (hybrid_available(n)) {
    while (!fpw.empty() && !lz.empty()) {  // wide fp64 primes first: more bits per walk
      gs.push_back(ModpGroup{2, true, 1, {lz.front(), fpw.front()}, false, true});
      lz.erase(lz.begin());
      fpw.erase(fpw.begin());
    }
    while (!fp.empty() && !lz.empty()) {
      gs.push_back(ModpGroup{2, true, 1, {lz.front(), fp.front()}});
      lz.erase(lz.begin());
      fp.erase(fp.begin());
    }
  }
  wd.insert(wd.end(), fpw.begin(), fpw.end());  // unpaired wide fp64 primes
  lz.insert(lz.end(), fp.begin(), fp.end());  // leftover small primes run as Montgomery
  for (int mode = 1; mode >= 0; --mode) {
    const std::vector<int>& sel = mode ? lz : red;
    size_t i = 0;
    while (i < sel.size()) {
      const int P = static_cast<int>(std::min<size_t>(pmax, sel.size() - i));
      ModpGroup g{P, mode == 1, 0, {}};
      for (int q = 0; q < P; ++q) g.idx.push_back(sel[i + q]);
      gs.push_back(g);
      i += P;
    }
  }
  const int wmax = kMaxPWide;
  for (size_t i = 0; i < wd.size();) {
    const int P = static_cast<int>(std::min<size_t>(wmax, wd.size() - i));
    ModpGroup g{P, false, 0, {}, true};
    for (int q = 0; q < P; ++q) g.idx.push_back(wd[i + q]);
    gs.push_back(g);
    i += P;
  }
  return gs;
}

}  // namespace pk

extern "C" int pk_ryser_modp(const uint64_t* a, const uint64_t* primes, int P, int n, int algo,
                             uint64_t start, uint64_t length, int ndev, uint64_t* out) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(P >= 0, kErrArg, "negative prime count");
    if (P == 0) return 0;
    PK_REQUIRE(a && primes && out, kErrArg, "null pointer argument");
    PK_REQUIRE(n >= 1, kErrArg, "empty matrix");
    PK_REQUIRE(algo == 0 || algo == 1, kErrArg, "algo must be 0 (ryser) or 1 (glynn)");
    PK_REQUIRE(n <= kBlockMaxN, kErrLimit, "dimension exceeds 64");
    const size_t nn = static_cast<size_t>(n) * n;
    for (int k = 0; k < P; ++k) {
      PK_REQUIRE(primes[k] >= 2 && primes[k] < (1ull << 62), kErrArg,
                 "modulus must be a prime in [2, 2^62)");
      for (size_t e = 0; e < nn; ++e)
        PK_REQUIRE(a[k * nn + e] < primes[k], kErrArg, "matrix residues must lie in [0, p)");
    }
    const Plan p = make_plan(n, algo);
    check_range(p.m, start, length);
    const Range r = make_range(p, start, length);
    const uint64_t nt = r.t1 - r.t0;
    std::vector<int> fast, slow;
    for (int k = 0; k < P; ++k) {
      if (walk_prime(primes[k]) && n <= kMaxN && nt > 0)
        fast.push_back(k);
      else
        slow.push_back(k);
    }
    std::vector<uint64_t> res(P, 0);
    const std::vector<ModpGroup> gs = group_primes(fast, primes, n);
    ndev = clamp_ndev(ndev);
    std::vector<uint64_t> cut(ndev + 1);
    for (int d = 0; d <= ndev; ++d) cut[d] = r.t0 + nt * d / ndev;
    std::vector<std::vector<uint64_t>> dev_res(ndev, std::vector<uint64_t>(P, 0));
    for_devices(ndev, [&](int d) {
      DevCtx& c = ctx(d);
      std::lock_guard<std::mutex> g(c.mu);
      PK_CUDA(cudaSetDevice(c.dev));
      const uint64_t t0 = cut[d], t1 = cut[d + 1];
      // fast kernels over the aligned interior, one launch per prime group
      for (size_t gi = 0; gi < gs.size() && t1 > t0; ++gi) {
        const ModpGroup& G = gs[gi];
        std::vector<uint64_t> gp;
        for (int k : G.idx) gp.push_back(primes[k]);
        const std::vector<uint8_t> ha = pack_residues(G, a, nn);
        void* d_a = c.a.get(ha.size());
        auto* d_o = static_cast<unsigned long long*>(c.modp_out.get(G.out_words() * 8));
        PK_CUDA(cudaMemcpyAsync(d_a, ha.data(), ha.size(), cudaMemcpyHostToDevice, c.stream));
        PK_CUDA(cudaMemsetAsync(d_o, 0, G.out_words() * 8, c.stream));
        ModpLaunch L = prepare_modp(c, p, G, algo, d_a, gp, t0, t1 - t0, d_o);
        launch_walk(c, L.fn, L.grid, L.smem, L.args);
        std::vector<unsigned long long> ho(G.out_words());
        PK_CUDA(cudaMemcpyAsync(ho.data(), d_o, ho.size() * 8, cudaMemcpyDeviceToHost, c.stream));
        PK_CUDA(cudaStreamSynchronize(c.stream));
        decode_group(G, ho.data(), primes, n, algo, dev_res[d].data());
      }
      // exact-kernel work, spread over the devices: the ragged head / tail
      // pieces of the fast primes round-robin, and every slow modulus (even,
      // composite or n > kMaxN) split into one contiguous share per device
      std::vector<std::pair<uint64_t, uint64_t>> ragged = r.head;
      ragged.insert(ragged.end(), r.tail.begin(), r.tail.end());
      auto* d_a = static_cast<uint64_t*>(c.a.get(nn * 8));
      for (int k = 0; k < P; ++k) {
        const bool is_fast = std::find(fast.begin(), fast.end(), k) != fast.end();
        std::vector<std::pair<uint64_t, uint64_t>> pcs;
        if (is_fast) {
          for (size_t i = d; i < ragged.size(); i += ndev) pcs.push_back(ragged[i]);
        } else {
          const uint64_t s0 = start + static_cast<uint64_t>(static_cast<u128>(length) * d / ndev);
          const uint64_t s1 = start + static_cast<uint64_t>(static_cast<u128>(length) * (d + 1) / ndev);
          // pieces of <= 2^(m-17) indices, and at least ~2^14 of them so that a
          // sub-range still fills the GPU (one thread walks one piece)
          const int lb = s1 > s0 ? 63 - __builtin_clzll(s1 - s0) : 0;
          const int bits = std::clamp(std::min(p.m - 17, lb - 14), 6, 62);
          split_pieces(s0, s1, bits, pcs);
        }
        if (pcs.empty()) continue;
        PK_CUDA(cudaMemcpyAsync(d_a, a + k * nn, nn * 8, cudaMemcpyHostToDevice, c.stream));
        const uint64_t v = modp_pieces(c, d_a, n, algo, primes[k], pcs);
        dev_res[d][k] = static_cast<uint64_t>((static_cast<u128>(dev_res[d][k]) + v) % primes[k]);
      }
    });
    for (int k = 0; k < P; ++k) {
      u128 s = 0;
      for (int d = 0; d < ndev; ++d) s += dev_res[d][k];
      out[k] = static_cast<uint64_t>(s % primes[k]);
    }
    return 0;
  });
}

// ---------------------------------------------------------------------------
// resident jobs

struct pk_job {
  int kind = 0;  // 0 f64, 1 modp
  DevCtx* c = nullptr;
  Plan plan;
  int algo = 0, n = 0, P = 0, B = 1, pf = 0;
  bool cplx = false;
  uint64_t t0 = 0, nt = 0;
  void* d_a = nullptr;
  double* d_part = nullptr;
  double* d_groups = nullptr;
  double* d_out = nullptr;
  uint32_t* d_primes = nullptr;
  unsigned long long* d_modp = nullptr;
  void* d_flush = nullptr;
  size_t flush_cap = 0;
  std::vector<uint64_t> prime_in;  // F_p: the caller's prime list (ModpGroup::idx refers to it)
  const void* fn = nullptr;
  int grid = 0, smem = 0, occ = 0;
  WalkArgs args{};
  std::vector<ModpLaunch> groups;  // F_p jobs: one launch per prime group
  std::vector<ModpGroup> gdesc;    // ... and its description (output words per group)
  size_t out_words = 0;            // F_p: length of d_modp
  std::vector<double> group_ms;    // F_p: per-group walk time of the last run
};

static void job_free(pk_job* j) {
  if (!j) return;
  if (j->c) cudaSetDevice(j->c->dev);
  cudaFree(j->d_a);
  cudaFree(j->d_part);
  cudaFree(j->d_groups);
  cudaFree(j->d_out);
  cudaFree(j->d_primes);
  cudaFree(j->d_modp);
  cudaFree(j->d_flush);
  delete j;
}

extern "C" int pk_job_f64_create(int device, const double* a, int n, int is_complex, int algo,
                                 uint64_t start, uint64_t length, pk_job** job) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(job != nullptr, kErrArg, "null job pointer");
    check_f64_args(a, n, algo);
    std::unique_ptr<pk_job, void (*)(pk_job*)> j(new pk_job, job_free);
    j->kind = 0;
    j->c = &ctx(device);
    DevCtx& c = *j->c;
    std::lock_guard<std::mutex> g(c.mu);
    PK_CUDA(cudaSetDevice(c.dev));
    j->plan = make_plan(n, algo);
    check_range(j->plan.m, start, length);
    const Range r = make_range(j->plan, start, length);
    PK_REQUIRE(r.head.empty() && r.tail.empty() && r.t1 > r.t0, kErrArg,
               "job range must be aligned to the tile span 2^(k+5)");
    j->algo = algo;
    j->n = n;
    j->cplx = is_complex != 0;
    j->t0 = r.t0;
    j->nt = r.t1 - r.t0;
    const size_t abytes = static_cast<size_t>(n) * n * (j->cplx ? 16 : 8);
    PK_CUDA(cudaMalloc(&j->d_a, abytes));
    PK_CUDA(cudaMemcpy(j->d_a, a, abytes, cudaMemcpyHostToDevice));
    PK_CUDA(cudaMalloc(&j->d_part, j->nt * kPartialStride * 8));
    PK_CUDA(cudaMalloc(&j->d_out, kPartialStride * 8));
    PK_CUDA(cudaMalloc(&j->d_groups, group_scratch_doubles(1, j->nt, j->plan.group) * 8));
    F64Launch L = prepare_f64(c, j->plan, j->cplx, algo, 1, static_cast<double*>(j->d_a), j->t0,
                              j->nt, false, j->d_part, a);
    j->fn = L.fn;
    j->grid = L.grid;
    j->smem = L.smem;
    j->occ = L.occ;
    j->args = L.args;
    *job = j.release();
    return 0;
  });
}

extern "C" int pk_job_modp_create(int device, const uint64_t* a, const uint64_t* primes, int P,
                                  int n, int algo, uint64_t start, uint64_t length, pk_job** job) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(job != nullptr && a && primes, kErrArg, "null pointer argument");
    PK_REQUIRE(P >= 1, kErrArg, "need at least one prime");
    PK_REQUIRE(n >= 1 && n <= kMaxN, kErrLimit, "dimension outside the GPU kernel range");
    std::unique_ptr<pk_job, void (*)(pk_job*)> j(new pk_job, job_free);
    j->kind = 1;
    j->c = &ctx(device);
    DevCtx& c = *j->c;
    std::lock_guard<std::mutex> g(c.mu);
    PK_CUDA(cudaSetDevice(c.dev));
    std::vector<int> fast;
    for (int k = 0; k < P; ++k) {
      PK_REQUIRE(walk_prime(primes[k]), kErrArg, "resident F_p jobs need odd moduli < 2^62");
      fast.push_back(k);
    }
    const std::vector<ModpGroup> gs = group_primes(fast, primes, n);
    j->plan = make_plan(n, algo);
    check_range(j->plan.m, start, length);
    const Range r = make_range(j->plan, start, length);
    PK_REQUIRE(r.head.empty() && r.tail.empty() && r.t1 > r.t0, kErrArg,
               "job range must be aligned to the tile span 2^(k+5)");
    j->algo = algo;
    j->n = n;
    j->P = P;
    j->B = static_cast<int>(gs.size());
    j->t0 = r.t0;
    j->nt = r.t1 - r.t0;
    const size_t nn = static_cast<size_t>(n) * n;
    std::vector<uint8_t> ha;
    std::vector<size_t> a_off, o_off;
    for (const auto& G : gs) {
      a_off.push_back(ha.size());
      o_off.push_back(j->out_words);
      const std::vector<uint8_t> g = pack_residues(G, a, nn);
      ha.insert(ha.end(), g.begin(), g.end());
      j->out_words += G.out_words();
    }
    PK_CUDA(cudaMalloc(&j->d_a, ha.size()));
    PK_CUDA(cudaMemcpy(j->d_a, ha.data(), ha.size(), cudaMemcpyHostToDevice));
    PK_CUDA(cudaMalloc(&j->d_modp, j->out_words * 8));
    for (size_t gi = 0; gi < gs.size(); ++gi) {
      const ModpGroup& G = gs[gi];
      std::vector<uint64_t> gp;
      for (int k : G.idx) gp.push_back(primes[k]);
      ModpLaunch L = prepare_modp(c, j->plan, G, algo, static_cast<uint8_t*>(j->d_a) + a_off[gi],
                                  gp, j->t0, j->nt, j->d_modp + o_off[gi]);
      j->groups.push_back(L);
      j->gdesc.push_back(G);
    }
    j->prime_in.assign(primes, primes + P);
    j->fn = j->groups.front().fn;
    j->grid = j->groups.front().grid;
    j->smem = j->groups.front().smem;
    j->occ = j->groups.front().occ;
    *job = j.release();
    return 0;
  });
}

extern "C" int pk_job_run(pk_job* j, int iters, size_t flush_bytes, double* total_ms,
                          double* walk_ms, double* out_f64, uint64_t* out_res) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(j != nullptr && iters >= 1, kErrArg, "bad job or iteration count");
    DevCtx& c = *j->c;
    std::lock_guard<std::mutex> g(c.mu);
    PK_CUDA(cudaSetDevice(c.dev));
    if (flush_bytes > j->flush_cap) {
      if (j->d_flush) PK_CUDA(cudaFree(j->d_flush));
      j->d_flush = nullptr;
      PK_CUDA(cudaMalloc(&j->d_flush, flush_bytes));
      j->flush_cap = flush_bytes;
    }
    // ev[0], ev[1]: the whole sequence; then per iteration one event before
    // each launch group and one after the last (F_p: G groups; f64: one)
    const int G = j->kind == 1 ? static_cast<int>(j->groups.size()) : 1;
    std::vector<cudaEvent_t> ev(2 + static_cast<size_t>(iters) * (G + 1));
    for (auto& e : ev) PK_CUDA(cudaEventCreate(&e));
    auto gev = [&](int it, int g) { return ev[2 + static_cast<size_t>(it) * (G + 1) + g]; };
    const size_t nres = j->kind == 1 ? j->out_words : 0;
    PK_CUDA(cudaEventRecord(ev[0], c.stream));
    for (int it = 0; it < iters; ++it) {
      if (flush_bytes) PK_CUDA(cudaMemsetAsync(j->d_flush, it & 0xff, flush_bytes, c.stream));
      if (j->kind == 1) PK_CUDA(cudaMemsetAsync(j->d_modp, 0, nres * 8, c.stream));
      if (j->kind == 0) {
        PK_CUDA(cudaEventRecord(gev(it, 0), c.stream));
        launch_walk(c, j->fn, j->grid, j->smem, j->args);
      } else {
        for (int g = 0; g < G; ++g) {
          PK_CUDA(cudaEventRecord(gev(it, g), c.stream));
          auto& L = j->groups[g];
          launch_walk(c, L.fn, L.grid, L.smem, L.args);
        }
      }
      PK_CUDA(cudaEventRecord(gev(it, G), c.stream));
      if (j->kind == 0)
        launch_reduce(c, j->d_part, 1, j->t0, j->nt, j->plan.group, j->d_groups, j->d_out);
    }
    PK_CUDA(cudaEventRecord(ev[1], c.stream));
    PK_CUDA(cudaEventSynchronize(ev[1]));
    float ms = 0;
    PK_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    if (total_ms) *total_ms = ms;
    double wsum = 0;
    j->group_ms.assign(G, 0.0);
    for (int it = 0; it < iters; ++it) {
      for (int g = 0; g < G; ++g) {
        PK_CUDA(cudaEventElapsedTime(&ms, gev(it, g), gev(it, g + 1)));
        j->group_ms[g] += ms;
        wsum += ms;
      }
    }
    if (walk_ms) *walk_ms = wsum;
    for (auto& e : ev) cudaEventDestroy(e);
    if (j->kind == 0 && out_f64)
      PK_CUDA(cudaMemcpy(out_f64, j->d_out, kPartialStride * 8, cudaMemcpyDeviceToHost));
    if (j->kind == 1 && out_res) {
      std::vector<unsigned long long> ho(nres);
      PK_CUDA(cudaMemcpy(ho.data(), j->d_modp, nres * 8, cudaMemcpyDeviceToHost));
      size_t s = 0;
      for (const ModpGroup& G : j->gdesc) {
        decode_group(G, ho.data() + s, j->prime_in.data(), j->n, j->algo, out_res);
        s += G.out_words();
      }
    }
    return 0;
  });
}

extern "C" int pk_job_info(pk_job* j, int64_t* info) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(j && info, kErrArg, "null argument");
    cudaFuncAttributes fa{};
    PK_CUDA(cudaSetDevice(j->c->dev));
    PK_CUDA(cudaFuncGetAttributes(&fa, j->fn));
    info[0] = j->plan.k;
    info[1] = static_cast<int64_t>(j->nt);
    info[2] = j->grid;
    info[3] = j->occ;
    info[4] = fa.numRegs;
    info[5] = static_cast<int64_t>(fa.localSizeBytes);
    info[6] = j->smem;
    info[7] = j->kind == 0 ? 3 : static_cast<int64_t>(j->groups.size());
    return 0;
  });
}

extern "C" int pk_job_groups(pk_job* j, int64_t* desc, double* ms, int64_t* prime_idx,
                             int max_groups) {
  return pk_guard([&]() -> int {
    PK_REQUIRE(j != nullptr, kErrArg, "null job");
    if (j->kind != 1) return 0;
    const int G = static_cast<int>(j->groups.size());
    PK_CUDA(cudaSetDevice(j->c->dev));
    for (int g = 0; g < std::min(G, max_groups); ++g) {
      const ModpGroup& D = j->gdesc[g];
      const ModpLaunch& L = j->groups[g];
      if (desc) {
        cudaFuncAttributes fa{};
        PK_CUDA(cudaFuncGetAttributes(&fa, L.fn));
        const int kind = D.wide ? 4 : D.pf ? (D.wf ? 3 : 2) : (D.lazy ? 1 : 0);
        const int64_t v[6] = {kind, D.P, fa.numRegs, L.occ, L.grid, L.smem};
        std::copy(v, v + 6, desc + 6 * g);
      }
      if (ms) ms[g] = g < static_cast<int>(j->group_ms.size()) ? j->group_ms[g] : 0.0;
      if (prime_idx)
        for (int q = 0; q < 4; ++q) prime_idx[4 * g + q] = q < D.P ? D.idx[q] : -1;
    }
    return G;
  });
}

extern "C" void pk_job_destroy(pk_job* j) { job_free(j); }
