// meshnbr.cu — host orchestration + C ABI of libmeshnbr.so (declared in include/meshnbr.h).
//
// mn_find_neighbors_both, fixed element types:
//   small meshes (<= 8192 incidences, <= 4096 nodes):   k_small_both, one CTA, one blocking read
//   otherwise:
//     k_locality_sample (+ 1 blocking read)   choose the element-CSR algorithm (meshes >= 2^20 elements)
//     element CSR, locality (config 5):       k_chunk_scatter_fixed (a1/a2 validation + one read of conn
//                                             into fixed 128-node chunk buckets, cursor atomics
//                                             pipelined across warp-blocks), k_scan_i32 (chunk bases),
//                                             guarded counted fallback, k_chunk_sort (a3e/a4/a5; bucket
//                                             read by TMA bulk copies)
//     element CSR, no locality (config 4):    k_hist_validate, k_bucket_bases, k_onesweep x nd (LSD,
//                                             pass 0 creates the pairs from conn, last pass writes the
//                                             payloads + run lengths), k_scan_i32 (a5)
//     node CSR:                               k_node_gather_t (a1/a3n/a4: per-node expansion of the
//                                             element CSR, hash-set dedupe, register sort), k_node_giant,
//                                             k_scan_i32 (a5)
//     k_read_words(err, nnz) + one stream sync a6 (a kernel store into pinned memory, not a D2H copy
//                                             that could queue behind a download on the copy engine)
//     exact-size node indices, k_node_compact  a6
// Host buffers: mn_find_neighbors_both_host (one call), mn_host_pipeline_* (a stream of meshes on
// three streams: the upload of mesh i+1 overlaps the download of mesh i).
// The paper-literal node pipeline (all node pairs, LSD over 2b key bits, k_unique_node) is
// mn_find_node_neighbors_sortpairs.  Polygons: poly.cuh; small meshes: small.cuh; multi-GPU:
// dist.cuh (bucket + NCCL all-to-all, or the fused bucket-and-send over peer memory).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"
#include "poly.cuh"
#include "small.cuh"

namespace mn {

// ================================================================================================
// instrumentation
// ================================================================================================
static std::atomic<int64_t> g_launches{0};
// element-CSR algorithm: 0 = auto (locality test), 1 = LSD radix sort, 2 = counting-sort transpose
static std::atomic<int> g_elem_path{0};
static std::atomic<int> g_chunk_cap{0};   // test knob: cap on the fixed chunk-bucket capacity (0 = auto)
static std::atomic<int64_t> g_small_max{kSmallMaxPe};   // incidences up to which the one-CTA path runs
constexpr int64_t kTransposeMinElems = 1 << 20;
constexpr int kMsdBins = 512;   // node ranges of the MSD element path
constexpr double kTransposeMaxGroupRatio = 0.5;
static bool g_prof = false;
struct ProfRec { const char* name; cudaEvent_t a, b; double bytes; };
static std::vector<ProfRec> g_recs;
static std::vector<cudaEvent_t> g_evpool;
struct ProfEntry { std::string name; int64_t launches; double ms; double bytes; };
static std::vector<ProfEntry> g_table;

static cudaEvent_t ev_get() {
  if (!g_evpool.empty()) { cudaEvent_t e = g_evpool.back(); g_evpool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// NVTX ranges (nvtx3, header-only: a no-op unless a tool such as ncu / nsys is attached): one per
// kernel launch (named as in the profiler table) and one per C-ABI entry point (NvtxScope).
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

template <class F>
static cudaError_t launch(const char* name, double alg_bytes, cudaStream_t s, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (g_prof) { a = ev_get(); b = ev_get(); cudaEventRecord(a, s); }
  const NvtxScope range(name);
  f();
  cudaError_t e = cudaGetLastError();
  if (g_prof) { cudaEventRecord(b, s); g_recs.push_back({name, a, b, alg_bytes}); }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return e;
}

// Adds bytes known only after the call's host sync (a list size) to the latest record of `name`.
// (skip: how many later records of the same name to pass over)
static void prof_add_bytes(const char* name, double bytes, int skip = 0) {
  if (!g_prof) return;
  for (auto it = g_recs.rbegin(); it != g_recs.rend(); ++it)
    if (std::strcmp(it->name, name) == 0 && skip-- == 0) { it->bytes += bytes; return; }
}

// ================================================================================================
// memory
// ================================================================================================
static void* default_alloc(void*, size_t bytes, mn_stream s) {
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, (cudaStream_t)s) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  return p;
}
static void default_release(void*, void* p, mn_stream s) {
  if (p) cudaFreeAsync(p, (cudaStream_t)s);
}
static const mn_allocator kDefaultAlloc = {default_alloc, default_release, nullptr};

struct Mem {
  mn_allocator a;
  cudaStream_t s;
  Mem(const mn_allocator* al, cudaStream_t st) : a(al && al->alloc ? *al : kDefaultAlloc), s(st) {}
  void* get(size_t bytes) { return a.alloc(a.ctx, bytes ? bytes : 16, (mn_stream)s); }
  void put(void* p) { if (p) a.release(a.ctx, p, (mn_stream)s); }
};

// Carves one workspace allocation into 256-byte aligned pieces (dry run with base == nullptr).
struct Arena {
  char* base = nullptr;
  size_t off = 0;
  template <typename X>
  X* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    // with base == nullptr the returned "pointer" is the byte offset (relocated by the caller)
    X* p = reinterpret_cast<X*>(reinterpret_cast<uintptr_t>(base) + off);
    off += count * sizeof(X);
    return p;
  }
};

// Per-thread pinned staging word pair for the one blocking read of (err, nnz).
static uint64_t* pinned_pair() {
  static thread_local uint64_t* p = nullptr;
  if (!p) {
    if (cudaMallocHost(&p, 4 * sizeof(uint64_t)) != cudaSuccess) { cudaGetLastError(); p = nullptr; }
  }
  return p;
}

// Per-device one-time setup (kernel attributes, occupancy-derived grids): one flag per (site,
// device), so a process that drives several GPUs, or several threads racing their first call, set
// every attribute on every device before its first launch there.
static int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); d = 0; }
  return d;
}
constexpr int kMaxDevices = 64;
struct PerDevice {
  std::mutex mu;
  bool done[kMaxDevices] = {};
  int value[kMaxDevices] = {};
  template <class F>
  int once(F&& f) {   // runs f() (returning int) once per device; returns its value for this device
    const int d = current_device();
    std::lock_guard<std::mutex> g(mu);
    if (d < 0 || d >= kMaxDevices) return f();
    if (!done[d]) { value[d] = f(); done[d] = true; }
    return value[d];
  }
};

// Small blocking readbacks (validation word, nnz, sample counts) are written into the pinned host
// words by a one-warp kernel, not a D2H copy: a copy would queue behind any large download on the
// device's D2H copy engine (the pipelined host API downloads the previous mesh's CSRs meanwhile:
// measured 68 ms instead of 9 for the call).  The host reads after the stream sync.
__global__ void k_read_words(const uint64_t* __restrict__ src, volatile uint64_t* dst, int n) {
  if ((int)threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}
static cudaError_t read_words(uint64_t* host_dst, const void* dev_src, int nbytes, cudaStream_t s) {
  k_read_words<<<1, 32, 0, s>>>(reinterpret_cast<const uint64_t*>(dev_src), host_dst, nbytes / 8);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

static mn_status decode_err(uint64_t w, mn_error_detail* err) {
  if (w == ERR_NONE) return MN_OK;
  if (err) { err->elem = (int64_t)(w >> 5); err->pos = (int32_t)(w & 15); }
  return ((w >> 4) & 1) ? MN_ERR_DEGENERATE : MN_ERR_INDEX_OUT_OF_RANGE;
}

#define MN_CUDA(x)                                        \
  do {                                                    \
    cudaError_t _e = (x);                                 \
    if (_e != cudaSuccess) { st = MN_ERR_CUDA; goto done; } \
  } while (0)

// ================================================================================================
// plans
// ================================================================================================
// onesweep pass tiles: 512 threads x 16 keys, 2 CTAs per SM, look-back window 4 (chosen with
// tools/sweep_onesweep.cu on B200: per-tile look-back cost dominates, so larger tiles win)
constexpr int kPassThreads = 512;
constexpr int kPassItems = 16;
constexpr int kPassMinBlocks = 2;
constexpr int kPassWindow = 4;
constexpr int kTile = kPassThreads * kPassItems;   // keys per onesweep tile
// compaction / scan tiles
constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kUTile = kThreads * kItems;
// single-pass scans: 1024 x 16 tiles (measured 0.39 vs 0.50 ms for config 5's two 33 M-entry scans
// with 256 x 16: fewer look-back steps)
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

// segment sort: 4096 staged entries (16 KB) and >= 8 CTAs per SM (64 registers): 2.17 ms on config 5
// vs 2.34 ms for 8192 entries / 78 registers (profiles/round1/sweep_segsort.txt)
static auto* const segsort_fn = &k_elem_segsort<4096, 8>;

struct Plan {
  int T, K, E, C;
  int64_t M, N;
  int b;
  bool key64;
  int bins;
  DigitPlan dp;
  int64_t Pn, Pe;
};

static DigitPlan make_digits(int bits, int* bins) {
  DigitPlan dp{};
  const int nd9 = (bits + 8) / 9, nd8 = (bits + 7) / 8;
  dp.nd = nd9;
  *bins = (nd8 == nd9) ? 256 : 512;
  int s = 0;
  for (int j = 0; j < dp.nd; ++j) {
    dp.width[j] = bits / dp.nd + (j < bits % dp.nd ? 1 : 0);
    dp.shift[j] = s;
    s += dp.width[j];
  }
  return dp;
}

static Plan make_plan(int T, int64_t M, int64_t N) {
  Plan P{};
  P.T = T; P.K = arity_of(T); P.E = edges_of(T); P.C = 2 * P.E / P.K;
  P.M = M; P.N = N;
  P.b = node_bits(N);
  P.key64 = 2 * P.b > 32;
  P.dp = make_digits(P.b, &P.bins);
  P.Pn = 2 * (int64_t)P.E * M;
  P.Pe = (int64_t)P.K * M;
  return P;
}

static int64_t tiles_of(int64_t n, int tile) { return (n + tile - 1) / tile; }
static int hist_grid(int64_t M) {
  int64_t g = (M + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  return g < 1 ? 1 : (int)g;
}
// the transpose count: a 2-wave grid (1.49 vs 1.55 ms on config 5); the scatter keeps hist_grid's
// single resident wave, which keeps its write window inside L2 (4 or 32 CTAs/SM: +40%)
static int count_grid(int64_t M) {
  int64_t g = (M + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}
static int stream_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

// ================================================================================================
// one onesweep pass
// ================================================================================================
template <typename KeyT, int SRC, int T, bool PAYLOAD, bool OWNER, int BINS, bool COUNTS = false>
static cudaError_t run_pass(PassArgs pa, cudaStream_t s, const char* name, double bytes) {
  using Sm = OnesweepSmem<kPassThreads, kPassItems, BINS>;
  const int64_t tiles = tiles_of(pa.n, kTile);
  if (tiles == 0) return cudaSuccess;
  const size_t smem = ((sizeof(Sm) + 15) & ~size_t(15)) + (size_t)kTile * sizeof(KeyT) +
                      ((PAYLOAD || SRC == 2) ? (size_t)kTile * 4 : 0);
  auto kern = k_onesweep<KeyT, SRC, T, PAYLOAD, OWNER, BINS, kPassThreads, kPassItems, kPassWindow, kPassMinBlocks,
                         0, COUNTS>;
  static PerDevice attr;
  attr.once([&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return 0;
  });
  return launch(name, bytes, s, [&] { kern<<<(unsigned)tiles, kPassThreads, smem, s>>>(pa); });
}

static PassDigit mask_digit(int shift, int width) {
  PassDigit pd{};
  pd.shift = shift;
  pd.mask = (1u << width) - 1u;
  pd.div = 1;
  return pd;
}

// ================================================================================================
// the whole path
// ================================================================================================
template <int T, typename KeyT, int BINS>
static mn_status pipeline(const Plan& P, const int32_t* conn, Mem& mem, bool want_node,
                          bool want_elem, mn_csr* node_out, mn_csr* elem_out,
                          mn_error_detail* err) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  const int nd = P.dp.nd;
  const int nnode_pass = want_node ? 2 * nd : 0;
  const int nelem_pass = want_elem ? nd : 0;
  const int npass = nnode_pass + nelem_pass;
  const int64_t node_tiles = tiles_of(P.Pn, kTile), elem_tiles = tiles_of(P.Pe, kTile);
  const int64_t st_tiles = std::max(want_node ? node_tiles : 0, want_elem ? elem_tiles : 0);
  const int64_t uq_tiles = want_node ? tiles_of(P.Pn, kUTile) : 0;
  const size_t w = sizeof(KeyT);
  // elem arrays alias the dead node key buffer when it is large enough
  const bool alias = want_node && want_elem && (size_t)P.Pn * w >= (size_t)16 * P.Pe;

  int64_t *node_off = nullptr, *elem_off = nullptr;
  int32_t *elem_idx = nullptr, *node_idx = nullptr;
  void* ws = nullptr;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;

  // ---- outputs known in size up front ----
  if (want_node) {
    node_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
    if (!node_off) { st = MN_ERR_OOM; goto done; }
  }
  if (want_elem) {
    elem_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
    elem_idx = P.Pe ? (int32_t*)mem.get((size_t)P.Pe * 4 + 16) : nullptr;
    if (!elem_off || (P.Pe && !elem_idx)) { st = MN_ERR_OOM; goto done; }
  }

  if (P.M == 0) {  // no pairs: every slice empty
    if (node_off) MN_CUDA(cudaMemsetAsync(node_off, 0, (size_t)(P.N + 1) * 8, s));
    if (elem_off) MN_CUDA(cudaMemsetAsync(elem_off, 0, (size_t)(P.N + 1) * 8, s));
    MN_CUDA(cudaStreamSynchronize(s));
    goto finish;
  }

  {
    // ---- workspace layout ----
    Arena ar;
    size_t head = 0;
    auto layout = [&](Arena& a, unsigned long long*& errw, unsigned long long*& nnz, uint32_t*& tickets,
                      unsigned long long*& hist, uint64_t*& bases, uint64_t*& status, uint64_t*& ustatus,
                      KeyT*& kA, KeyT*& kB, uint32_t*& ekA, uint32_t*& ekB, uint32_t*& epA, uint32_t*& epB) {
      errw = a.take<unsigned long long>(2);   // [0] validation word, [1] node nnz (one D2H read)
      nnz = errw + 1;
      tickets = a.take<uint32_t>(32);
      hist = a.take<unsigned long long>((size_t)nd * BINS);
      bases = a.take<uint64_t>((size_t)(npass ? npass : 1) * BINS);
      status = a.take<uint64_t>((size_t)st_tiles * BINS);
      ustatus = a.take<uint64_t>((size_t)(uq_tiles ? uq_tiles : 1));
      head = a.off;   // everything above is zero-initialised once per call
      kA = kB = nullptr;
      ekA = ekB = epA = epB = nullptr;
      if (want_node) { kA = a.take<KeyT>(P.Pn); kB = a.take<KeyT>(P.Pn); }
      if (want_elem) {
        if (alias && kB) {
          uint32_t* r = reinterpret_cast<uint32_t*>(kB);
          ekA = r; ekB = r + P.Pe; epA = r + 2 * P.Pe; epB = r + 3 * P.Pe;
        } else {
          ekA = a.take<uint32_t>(P.Pe); ekB = a.take<uint32_t>(P.Pe);
          epA = a.take<uint32_t>(P.Pe); epB = a.take<uint32_t>(P.Pe);
        }
      }
    };
    unsigned long long *errw, *nnz, *hist;
    uint32_t* tickets;
    uint64_t *bases, *status, *ustatus;
    KeyT *kA, *kB;
    uint32_t *ekA, *ekB, *epA, *epB;
    layout(ar, errw, nnz, tickets, hist, bases, status, ustatus, kA, kB, ekA, ekB, epA, epB);
    ws = mem.get(ar.off);
    if (!ws) { st = MN_ERR_OOM; goto done; }
    ar = Arena{};
    ar.base = (char*)ws;
    layout(ar, errw, nnz, tickets, hist, bases, status, ustatus, kA, kB, ekA, ekB, epA, epB);

    MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
    MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));

    // ---- a1/a2: validate + histograms ----
    MN_CUDA(launch("hist_validate", 4.0 * P.K * P.M, s, [&] {
      if (((uintptr_t)conn & 15) == 0)
        k_hist_validate<T, BINS, true><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, 0, P.dp, 0, 1, hist, errw);
      else
        k_hist_validate<T, BINS, false><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, 0, P.dp, 0, 1, hist, errw);
    }));
    BasesDesc bd{};
    bd.npass = npass;
    for (int q = 0; q < nnode_pass; ++q) { bd.hidx[q] = q % nd; bd.mult[q] = P.C; }
    for (int q = 0; q < nelem_pass; ++q) { bd.hidx[nnode_pass + q] = q; bd.mult[nnode_pass + q] = 1; }
    MN_CUDA(launch("bucket_bases", 0.0, s, [&] {
      k_bucket_bases<BINS><<<npass, BINS, 0, s>>>(hist, bd, bases, errw);
    }));

    uint32_t epoch = 0;
    // ---- a1 + a3n: node pairs, LSD over v digits then a digits ----
    if (want_node) {
      KeyT* in = nullptr;
      KeyT* bufs[2] = {kA, kB};
      for (int q = 0; q < nnode_pass; ++q) {
        const int j = q % nd;
        const int shift = (q < nd ? 0 : P.b) + P.dp.shift[j];
        PassArgs pa{};
        pa.keys_in = in;
        pa.keys_out = bufs[q & 1];
        pa.conn = conn;
        pa.node_bits = P.b;
        pa.n = P.Pn;
        pa.pd = mask_digit(shift, P.dp.width[j]);
        pa.bases = bases + (size_t)q * BINS;
        pa.status = status;
        pa.ticket = tickets + q;
        pa.epoch = ++epoch;
        pa.err = errw;
        if (q == 0) {
          MN_CUDA((run_pass<KeyT, 1, T, false, false, BINS>(pa, s, "onesweep_node_first",
                                                             4.0 * P.K * P.M + (double)w * P.Pn)));
        } else {
          MN_CUDA((run_pass<KeyT, 0, 0, false, false, BINS>(pa, s, "onesweep_node", 2.0 * w * P.Pn)));
        }
        in = bufs[q & 1];
      }
      // ---- a4 + a5: dedupe, compaction, run lengths, offsets ----
      UniqueArgs ua{};
      ua.keys = in;
      ua.n = P.Pn;
      ua.b = P.b;
      ua.N = P.N;
      ua.offsets = node_off;
      ua.indices = reinterpret_cast<uint32_t*>(in == kA ? kB : kA);
      ua.status = ustatus;
      ua.ticket = tickets + 30;
      ua.epoch = 1;
      ua.nnz = nnz;
      ua.err = errw;
      MN_CUDA(launch("unique_node", (double)w * P.Pn + 8.0 * (P.N + 1), s, [&] {
        k_unique_node<KeyT, kThreads, kItems><<<(unsigned)uq_tiles, kThreads, 0, s>>>(ua);
      }));
      node_idx = reinterpret_cast<int32_t*>(ua.indices);
    }

    // ---- a2 + a3e: element pairs, stable LSD over the node digits ----
    if (want_elem) {
      uint32_t* kb[2] = {ekA, ekB};
      uint32_t* vb[2] = {epA, epB};
      const uint32_t* kin = nullptr;
      const uint32_t* vin = nullptr;
      for (int q = 0; q < nelem_pass; ++q) {
        PassArgs pa{};
        pa.keys_in = kin;
        pa.vals_in = vin;
        pa.keys_out = kb[q & 1];
        pa.vals_out = (q == nelem_pass - 1) ? reinterpret_cast<uint32_t*>(elem_idx) : vb[q & 1];
        pa.conn = conn;
        pa.n = P.Pe;
        pa.pd = mask_digit(P.dp.shift[q], P.dp.width[q]);
        pa.bases = bases + (size_t)(nnode_pass + q) * BINS;
        pa.status = status;
        pa.ticket = tickets + 16 + q;
        pa.epoch = ++epoch;
        pa.err = errw;
        if (q == 0) {
          MN_CUDA((run_pass<uint32_t, 2, T, false, false, BINS>(pa, s, "onesweep_elem_first",
                                                                 4.0 * P.Pe + 8.0 * P.Pe)));
        } else {
          MN_CUDA((run_pass<uint32_t, 0, 0, true, false, BINS>(pa, s, "onesweep_elem", 16.0 * P.Pe)));
        }
        kin = kb[q & 1];
        vin = vb[q & 1];
      }
      MN_CUDA(launch("elem_offsets", 4.0 * P.Pe + 8.0 * (P.N + 1), s, [&] {
        k_elem_offsets<false><<<stream_grid(P.Pe / 4 + 1), 256, 0, s>>>(kin, P.Pe, P.N, elem_off, errw);
      }));
    }

    // ---- a6: one blocking read of (err, nnz) ----
    MN_CUDA(read_words(host, errw, 16, s));
    MN_CUDA(cudaStreamSynchronize(s));
    st = decode_err(host[0], err);
    if (st != MN_OK) goto done;
    if (want_node) {
      const int64_t U = (int64_t)host[1];
      int32_t* out = U ? (int32_t*)mem.get((size_t)U * 4) : nullptr;
      if (U && !out) { st = MN_ERR_OOM; goto done; }
      if (U) MN_CUDA(cudaMemcpyAsync(out, node_idx, (size_t)U * 4, cudaMemcpyDeviceToDevice, s));
      node_out->nnz = U;
      node_out->indices = out;
      node_idx = out;
    }
  }

finish:
  if (want_node) {
    node_out->num_nodes = P.N;
    node_out->offsets = node_off;
    if (P.M == 0) { node_out->nnz = 0; node_out->indices = nullptr; }
    node_out->owner = mem.a;
  }
  if (want_elem) {
    elem_out->num_nodes = P.N;
    elem_out->offsets = elem_off;
    elem_out->nnz = P.Pe;
    elem_out->indices = elem_idx;
    elem_out->owner = mem.a;
  }
  mem.put(ws);
  return MN_OK;

done:
  if (ws) { cudaStreamSynchronize(s); mem.put(ws); }
  mem.put(node_off);
  mem.put(elem_off);
  mem.put(elem_idx);
  if (want_node && node_out) { std::memset(node_out, 0, sizeof(*node_out)); }
  if (want_elem && elem_out) { std::memset(elem_out, 0, sizeof(*elem_out)); }
  return st;
}

// ================================================================================================
// the whole path, B200 restructure (DESIGN.md §"Node path"): element pairs are radix-sorted once
// (stable, node digits); the element CSR falls out of it and the node CSR is the per-node
// expansion of the element CSR (C edge-neighbours per incidence), sorted and deduplicated per
// node, counted, scanned, and compacted into an exact-size output after the one host sync.
// ================================================================================================
// Host-buffer calls: the element CSR is copied to the host on a side stream as soon as it is
// complete, overlapping the node pass (its sizes are known up front; the node CSR's are not).
struct HostSink {
  int64_t* h_elem_off;
  int32_t* h_elem_idx;
  cudaStream_t side;
  cudaEvent_t ev;
  bool issued;
};

template <int T, int BINS>
static mn_status pipeline_inc(const Plan& P, const int32_t* conn, Mem& mem, bool want_node, bool want_elem,
                              mn_csr* node_out, mn_csr* elem_out, mn_error_detail* err, HostSink* sink = nullptr,
                              bool shared = false) {
  const int CE = shared ? P.K - 1 : P.C;   // node candidates per incidence (node raw region: CE * Pe)
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  const int nd = P.dp.nd;
  const int64_t elem_tiles = tiles_of(P.Pe, kTile);
  const int64_t scan_tiles = tiles_of(P.N, kScanTile);
  const int64_t giant_cap = P.N;   // any node may overflow the warp path (> 32 distinct neighbours)
  const bool aligned = ((uintptr_t)conn & 15) == 0;
  bool transpose = false;
  bool msd = false;   // MSD element path (node-range buckets + CTA-local finish)
  const int64_t msd_R = (P.N + kMsdBins - 1) / kMsdBins;
  int64_t *node_off = nullptr, *elem_off = nullptr;
  int32_t* elem_idx = nullptr;
  void* ws = nullptr;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;

  // ---- outputs known in size up front ----
  if (want_node) {
    node_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
    if (!node_off) { st = MN_ERR_OOM; goto done; }
  }
  if (want_elem) {
    elem_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
    elem_idx = P.Pe ? (int32_t*)mem.get((size_t)P.Pe * 4 + 16) : nullptr;
    if (!elem_off || (P.Pe && !elem_idx)) { st = MN_ERR_OOM; goto done; }
  }
  if (P.M == 0) {
    if (node_off) MN_CUDA(cudaMemsetAsync(node_off, 0, (size_t)(P.N + 1) * 8, s));
    if (elem_off) MN_CUDA(cudaMemsetAsync(elem_off, 0, (size_t)(P.N + 1) * 8, s));
    MN_CUDA(cudaStreamSynchronize(s));
    if (want_node) { node_out->num_nodes = P.N; node_out->nnz = 0; node_out->offsets = node_off; node_out->indices = nullptr; node_out->owner = mem.a; }
    if (want_elem) { elem_out->num_nodes = P.N; elem_out->nnz = 0; elem_out->offsets = elem_off; elem_out->indices = nullptr; elem_out->owner = mem.a; }
    return MN_OK;
  }
  // ---- element-CSR algorithm: transpose when consecutive elements share nodes (locality) ----
  {
    const int mode = g_elem_path.load();
    if (mode == 2) {
      transpose = true;
    } else if (mode == 0 && P.M >= kTransposeMinElems) {
      unsigned long long* smp = (unsigned long long*)mem.get(16);
      if (!smp) { st = MN_ERR_OOM; goto done; }
      MN_CUDA(cudaMemsetAsync(smp, 0, 16, s));
      MN_CUDA(launch("locality_sample", 0.0, s, [&] {
        if (aligned) k_locality_sample<T, true><<<64, 256, 0, s>>>(conn, P.M, smp);
        else k_locality_sample<T, false><<<64, 256, 0, s>>>(conn, P.M, smp);
      }));
      MN_CUDA(read_words(host + 2, smp, 16, s));
      MN_CUDA(cudaStreamSynchronize(s));
      mem.put(smp);
      transpose = host[3] > 0 && (double)host[2] < kTransposeMaxGroupRatio * (double)host[3];
    }
  }
  // element CSR without the transpose: MSD bucketing by node range + CTA-local finish when each of
  // the 512 ranges fits in shared memory, else the LSD radix sort
  {
    const int epm = g_elem_path.load();
    // (not chosen in auto mode: on config 4 hist 0.19 + bucketing pass 1.45 + range finish 2.67 ms
    // vs 4.13 ms for the three LSD passes -- the scatter of element ids inside each range is random
    // 4-byte writes, 7x write amplification in DRAM when the windows leave L2)
    msd = !transpose && P.M > 0 && msd_R >= 1 && msd_R <= kRangeMax && epm == 3;
  }
  {
    // ---- workspace ----
    size_t head = 0;
    unsigned long long *errw = nullptr, *hist = nullptr;
    uint32_t *tickets = nullptr, *ekA = nullptr, *ekB = nullptr, *epA = nullptr, *epB = nullptr, *giants = nullptr;
    unsigned int* ngiant = nullptr;
    uint64_t *bases = nullptr, *status = nullptr, *sstatus = nullptr;
    int32_t *cnt = nullptr, *ecnt = nullptr, *lofs = nullptr, *cursor = nullptr;
    int32_t* ncsum = nullptr;   // per 128-node chunk: node-list total (k_node_gather_t, k_node_giant)
    int64_t* ncb = nullptr;     // its exclusive scan: the chunks' node-CSR bases
    uint32_t* sgiants = nullptr;
    unsigned int* nsgiant = nullptr;
    int64_t* eoff = elem_off;
    int32_t* eidx = elem_idx;
    const int64_t nchunks = tiles_of(P.N, kChunkNodes);
    int32_t *ccnt = nullptr, *ccur = nullptr;
    unsigned int* ovf = nullptr;   // a fixed-capacity chunk bucket overflowed
    unsigned long long* mhist = nullptr;   // MSD path: per-range incidence counts, bases, status
    uint64_t *mbases = nullptr, *mstatus = nullptr;
    int64_t* cbase = nullptr;
    auto layout = [&](Arena& a) {
      errw = a.take<unsigned long long>(2);
      tickets = a.take<uint32_t>(32);
      ngiant = a.take<unsigned int>(1);
      hist = a.take<unsigned long long>((size_t)nd * BINS);
      bases = a.take<uint64_t>((size_t)nd * BINS);
      status = a.take<uint64_t>((size_t)elem_tiles * BINS);
      sstatus = a.take<uint64_t>((size_t)(scan_tiles ? scan_tiles : 1));
      ecnt = a.take<int32_t>((size_t)P.N + 1);   // per-node incidence counts (atomics in the last pass)
      nsgiant = a.take<unsigned int>(1);
      if (transpose) cursor = a.take<int32_t>((size_t)P.N + 1);
      if (transpose) {
        ccnt = a.take<int32_t>((size_t)nchunks + 1);
        ccur = a.take<int32_t>((size_t)nchunks + 1);
        ovf = a.take<unsigned int>(1);
      }
      if (msd) {
        mhist = a.take<unsigned long long>(kMsdBins);
        mstatus = a.take<uint64_t>((size_t)(elem_tiles ? elem_tiles : 1) * kMsdBins);
      }
      head = a.off;
      if (msd) mbases = a.take<uint64_t>(kMsdBins);
      if (transpose || msd) sgiants = a.take<uint32_t>((size_t)P.N + 1);
      if (transpose) cbase = a.take<int64_t>((size_t)nchunks + 1);
      // ekA | ekB | epA | epB (each 256-byte aligned, contiguous); later the node raw region
      ekA = a.take<uint32_t>((size_t)P.Pe * (CE > 4 ? CE - 3 : 1));   // the 4 pieces hold >= CE * Pe
      ekB = a.take<uint32_t>((size_t)P.Pe);
      epA = a.take<uint32_t>((size_t)P.Pe);
      epB = a.take<uint32_t>((size_t)P.Pe);
      if (want_node) {
        cnt = a.take<int32_t>((size_t)P.N);
        lofs = a.take<int32_t>((size_t)P.N);
        ncsum = a.take<int32_t>((size_t)tiles_of(P.N, kNodeThreads) + 1);
        ncb = a.take<int64_t>((size_t)tiles_of(P.N, kNodeThreads) + 1);
        giants = a.take<uint32_t>((size_t)(giant_cap ? giant_cap : 1));
        if (!want_elem) {
          eoff = a.take<int64_t>((size_t)P.N + 1);
          eidx = a.take<int32_t>((size_t)P.Pe + 4);
        }
      }
    };
    Arena ar;
    layout(ar);
    ws = mem.get(ar.off);
    if (!ws) { st = MN_ERR_OOM; goto done; }
    ar = Arena{};
    ar.base = (char*)ws;
    eoff = elem_off;
    eidx = elem_idx;
    layout(ar);
    MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
    MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));

    const int scap = 48 * 1024;
    static PerDevice seg_attr;
    seg_attr.once([&] {
      cudaFuncSetAttribute(k_segsort_giant, cudaFuncAttributeMaxDynamicSharedMemorySize, scap * 4);
      return 0;
    });
    if (transpose) {
      // ---- a2 + a3e + a4 + a5 (elements): transpose bucketed by 128-node chunk ----
      // belem spans ekA + ekB (>= 2 Pe entries), bnode the bytes of epA + epB (>= 8 Pe)
      int32_t* belem = reinterpret_cast<int32_t*>(ekA);
      uint8_t* bnode = reinterpret_cast<uint8_t*>(epA);
      // single conn read: fixed-capacity buckets of cap entries (2 Pe / nchunks, i.e. twice the mean
      // chunk load); on overflow the counted path below runs (guarded by *ovf) and replaces it
      int64_t capl = nchunks > 0 ? (2 * P.Pe / nchunks) & ~(int64_t)31 : 0;
      const int ovr = g_chunk_cap.load();
      if (ovr > 0 && ovr < capl) capl = ovr;
      if (capl > (int64_t)INT32_MAX - 4096) capl = (int64_t)INT32_MAX - 4096;
      const int cap = (int)capl;
      // grid-stride over 256-thread CTAs, 4 per SM (3 for meshes of >= 2^26 elements): the grid sets
      // how wide the element window in flight is; wider (5-6 CTAs per SM, the occupancy limit at 40
      // registers) measured slower on config 5 (2.47 / 2.64 ms vs 2.14 at 4 and 2.07 at 3; 2 CTAs:
      // 2.72), config 3 is fastest at 4 (0.157 ms vs 0.165 at 3)
      // (never more than are resident at once: hex rows need 106 registers, 2 CTAs per SM)
      static PerDevice sm_count, occ_scatter;
      const int sms = sm_count.once([&] {
        int n = 148;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
        return n;
      });
      const int occ = occ_scatter.once([&] {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_chunk_scatter_fixed<T, true>, 256, 0);
        return o > 0 ? o : 1;
      });
      const int64_t fixed_wave = (int64_t)std::min(P.M >= ((int64_t)1 << 26) ? 3 : 4, occ) * sms;
      const int fgrid = (int)std::min<int64_t>(fixed_wave, (P.M + 255) / 256 > 0 ? (P.M + 255) / 256 : 1);
      MN_CUDA(launch("elem_scatter", 4.0 * P.K * P.M + 5.0 * P.Pe, s, [&] {
        if (aligned)
          k_chunk_scatter_fixed<T, true><<<fgrid, 256, 0, s>>>(conn, P.M, P.N, cap, ccur, belem, bnode, errw, ovf);
        else
          k_chunk_scatter_fixed<T, false><<<fgrid, 256, 0, s>>>(conn, P.M, P.N, cap, ccur, belem, bnode, errw, ovf);
      }));
      if (nchunks > 0)
        MN_CUDA(launch("scan_counts", 12.0 * nchunks, s, [&] {
          k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nchunks, kScanTile), kScanThreads, 0, s>>>(
              ccur, nchunks, cbase, sstatus, tickets + 29, 1);
        }));
      // ---- fallback (only if a bucket overflowed; otherwise each kernel returns at once) ----
      MN_CUDA(launch("count_fallback", 0.0, s, [&] {
        if (aligned)
          k_chunk_count<T, true><<<count_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, ccnt, errw, 0, INT64_MAX, ovf);
        else
          k_chunk_count<T, false><<<count_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, ccnt, errw, 0, INT64_MAX, ovf);
      }));
      if (nchunks > 0)
        MN_CUDA(launch("scan_fallback", 0.0, s, [&] {
          k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nchunks, kScanTile), kScanThreads, 0, s>>>(
              ccnt, nchunks, cbase, sstatus, tickets + 28, 3, ovf);
        }));
      MN_CUDA(launch("scatter_fallback", 0.0, s, [&] {
        if (aligned)
          k_chunk_scatter<T, true><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, cbase, cursor, belem, bnode, errw,
                                                                   0, INT64_MAX, ovf);
        else
          k_chunk_scatter<T, false><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, cbase, cursor, belem, bnode, errw,
                                                                    0, INT64_MAX, ovf);
      }));
      if (nchunks > 0)
        MN_CUDA(launch("elem_segsort", 9.0 * P.Pe + 8.0 * (P.N + 1), s, [&] {
          // sorted even for node-only calls: the gather then visits each node's element rows in
          // ascending order (L1 reuse; config 5 element-sharing CSR: gather 5.38 -> 4.13 ms for
          // +0.77 ms of sorting, step 10.28 -> 9.78 ms)
          k_chunk_sort<true><<<(unsigned)nchunks, kChunkNodes, 0, s>>>(cbase, P.N, belem, bnode, eoff, eidx,
                                                                        sgiants, nsgiant, errw, ovf, cap);
        }));
      if (want_elem)
        MN_CUDA(launch("segsort_giant", 0.0, s, [&] {
          k_segsort_giant<<<148, 1024, scap * 4, s>>>(eoff, eidx, sgiants, nsgiant, scap, errw);
        }));
    } else if (msd) {
      // ---- a2 + a3e + a4 + a5 (elements), MSD: stable bucketing by node range, CTA-local finish ----
      MN_CUDA(launch("hist_validate", 4.0 * P.K * P.M, s, [&] {
        if (aligned)
          k_hist_validate<T, kMsdBins, true><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, 0, P.dp, 1,
                                                                            (uint64_t)msd_R, mhist, errw);
        else
          k_hist_validate<T, kMsdBins, false><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, 0, P.dp, 1,
                                                                             (uint64_t)msd_R, mhist, errw);
      }));
      BasesDesc bd{};
      bd.npass = 1;
      bd.hidx[0] = 0;
      bd.mult[0] = 1;
      MN_CUDA(launch("bucket_bases", 0.0, s, [&] {
        k_bucket_bases<kMsdBins><<<1, kMsdBins, 0, s>>>(mhist, bd, mbases, errw);
      }));
      PassArgs pa{};
      pa.keys_out = ekA;
      pa.vals_out = epA;
      pa.conn = conn;
      pa.n = P.Pe;
      pa.pd.shift = 0;
      pa.pd.div = (uint64_t)msd_R;
      pa.pd.mask = 0;
      pa.bases = mbases;
      pa.status = mstatus;
      pa.ticket = tickets;
      pa.epoch = 1;
      pa.err = errw;
      MN_CUDA((run_pass<uint32_t, 2, T, false, true, kMsdBins>(pa, s, "onesweep_elem_first", 12.0 * P.Pe)));
      const size_t rsm = (size_t)msd_R * 4;
      static PerDevice rattr;
      rattr.once([&] {
        cudaFuncSetAttribute(k_range_transpose<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRangeMax * 4);
        return 0;
      });
      // persistent grid of 96 CTAs (one per SM at most): their random-write windows (one bucket's
      // element ids, 1 MB each on config 4) stay in L2.  Config 4: 3.72 ms with 512 CTAs, 3.92 with
      // 148, 2.67 with 96, 3.00 with 64, 4.65 with 40.
      const unsigned rgrid = 96;
      MN_CUDA(launch("range_transpose", 8.0 * P.Pe + 4.0 * P.Pe + 8.0 * (P.N + 1), s, [&] {
        // sorted also for node-only calls (ascending element-row visits in the gather)
        k_range_transpose<true><<<rgrid, kRangeThreads, rsm, s>>>(ekA, epA, mbases, kMsdBins, (int)msd_R, P.N,
                                                                     P.Pe, eoff, eidx, sgiants, nsgiant, errw);
      }));
      if (want_elem)
        MN_CUDA(launch("segsort_giant", 0.0, s, [&] {
          k_segsort_giant<<<148, 1024, scap * 4, s>>>(eoff, eidx, sgiants, nsgiant, scap, errw);
        }));
    } else {
    // ---- a1/a2 validation + digit histograms of the node ids ----
    MN_CUDA(launch("hist_validate", 4.0 * P.K * P.M, s, [&] {
      if (((uintptr_t)conn & 15) == 0)
        k_hist_validate<T, BINS, true><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, 0, P.dp, 0, 1, hist, errw);
      else
        k_hist_validate<T, BINS, false><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, 0, P.dp, 0, 1, hist, errw);
    }));
    BasesDesc bd{};
    bd.npass = nd;
    for (int q = 0; q < nd; ++q) { bd.hidx[q] = q; bd.mult[q] = 1; }
    MN_CUDA(launch("bucket_bases", 0.0, s, [&] { k_bucket_bases<BINS><<<nd, BINS, 0, s>>>(hist, bd, bases, errw); }));

    // ---- a2 + a3: element pairs (node, element) created from conn, stable LSD on the node digits ----
    uint32_t* kb[2] = {ekA, ekB};
    uint32_t* vb[2] = {epA, epB};
    const uint32_t* kin = nullptr;
    const uint32_t* vin = nullptr;
    // The last pass writes only the payloads (the element-CSR indices, in place) and adds each
    // node's run lengths to ecnt (a4: reduction of the ones array).
    for (int q = 0; q < nd; ++q) {
      const bool last = q == nd - 1;
      PassArgs pa{};
      pa.keys_in = kin;
      pa.vals_in = vin;
      pa.keys_out = last ? nullptr : kb[q & 1];
      pa.vals_out = last ? reinterpret_cast<uint32_t*>(eidx) : vb[q & 1];
      pa.conn = conn;
      pa.n = P.Pe;
      pa.pd = mask_digit(P.dp.shift[q], P.dp.width[q]);
      pa.bases = bases + (size_t)q * BINS;
      pa.status = status;
      pa.ticket = tickets + q;
      pa.epoch = (uint32_t)(q + 1);
      pa.err = errw;
      pa.counts = ecnt;
      if (q == 0 && !last) {
        MN_CUDA((run_pass<uint32_t, 2, T, false, false, BINS>(pa, s, "onesweep_elem_first", 12.0 * P.Pe)));
      } else if (q == 0) {
        MN_CUDA((run_pass<uint32_t, 2, T, false, false, BINS, true>(pa, s, "onesweep_elem_first", 8.0 * P.Pe)));
      } else if (!last) {
        MN_CUDA((run_pass<uint32_t, 0, 0, true, false, BINS>(pa, s, "onesweep_elem", 16.0 * P.Pe)));
      } else {
        MN_CUDA((run_pass<uint32_t, 0, 0, true, false, BINS, true>(pa, s, "onesweep_elem_last", 12.0 * P.Pe)));
      }
      kin = kb[q & 1];
      vin = vb[q & 1];
    }
    // ---- a5 (elements): exclusive scan of the per-node counts -> offsets ----
    if (P.N > 0)
      MN_CUDA(launch("scan_counts", 4.0 * P.N + 8.0 * (P.N + 1), s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)scan_tiles, kScanThreads, 0, s>>>(ecnt, P.N, eoff, sstatus,
                                                                                 tickets + 29, 1);
      }));
    }   // LSD element path

    if (sink && want_elem) {   // element CSR complete: stream it to the host during the node pass
      MN_CUDA(cudaEventRecord(sink->ev, s));
      MN_CUDA(cudaStreamWaitEvent(sink->side, sink->ev, 0));
      MN_CUDA(cudaMemcpyAsync(sink->h_elem_off, eoff, (size_t)(P.N + 1) * 8, cudaMemcpyDeviceToHost, sink->side));
      if (P.Pe)
        MN_CUDA(cudaMemcpyAsync(sink->h_elem_idx, eidx, (size_t)P.Pe * 4, cudaMemcpyDeviceToHost, sink->side));
      sink->issued = true;
    }
    int64_t U = 0;
    if (want_node) {
      // ---- a1 + a3n + a4 (nodes): expand the element CSR per node, sort + dedupe per node ----
      uint32_t* temp = ekA;   // CE * Pe entries: the dead element-sort buffers (ekA widened when CE > 4)
      // algorithmic bytes: element-CSR offsets + indices, every connectivity row once, counts and
      // list offsets written; the written lists (4 B per distinct neighbour) are added after the sync
      const double gb = 8.0 * (P.N + 1) + 4.0 * P.Pe + 4.0 * P.K * P.M + 8.0 * P.N;
      const unsigned ng = (unsigned)tiles_of(P.N, kNodeThreads);
      if (P.N > 0) {   // (M > 0 with N == 0 always fails validation: nothing to expand)
        MN_CUDA(launch("node_gather", gb, s, [&] {
          const RowSrc rs{conn, 0, P.M, nullptr, nullptr, 0};
          // meshes without locality (the LSD element path) gather their rows at random: those loads
          // fill 64 bytes of L2 instead of the default 128 (config 4: DRAM 15.4 -> 8.7 GB per launch; time
          // 2.57 -> 2.42 ms in one A/B, 2.61-2.63 on another box: the kernel is latency-bound there)
          if (shared && aligned && !transpose)
            k_node_gather_t<T, true, false, true, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, P.N, temp, cnt,
                                                                                   lofs, giants, ngiant, errw, 0, ncsum);
          else if (shared && aligned)
            k_node_gather_t<T, true, false, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, P.N, temp, cnt, lofs,
                                                                              giants, ngiant, errw, 0, ncsum);
          else if (shared)
            k_node_gather_t<T, false, false, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, P.N, temp, cnt, lofs,
                                                                               giants, ngiant, errw, 0, ncsum);
          else if (aligned && !transpose)
            k_node_gather_t<T, true, false, false, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, P.N, temp, cnt,
                                                                                    lofs, giants, ngiant, errw, 0, ncsum);
          else if (aligned)
            k_node_gather_t<T, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, P.N, temp, cnt, lofs, giants,
                                                                 ngiant, errw, 0, ncsum);
          else
            k_node_gather_t<T, false><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, P.N, temp, cnt, lofs, giants,
                                                                  ngiant, errw, 0, ncsum);
        }));
      }
      const int cap = 48 * 1024;   // uint32 entries sorted in shared memory by k_node_giant (192 KB)
      static PerDevice giant_attr;
      giant_attr.once([&] {
        cudaFuncSetAttribute(k_node_giant<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
        cudaFuncSetAttribute(k_node_giant<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
        cudaFuncSetAttribute(k_node_giant<T, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
        cudaFuncSetAttribute(k_node_giant<T, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
        return 0;
      });
      MN_CUDA(launch("node_giant", 0.0, s, [&] {
        const RowSrc rs{conn, 0, P.M, nullptr, nullptr, 0};
        if (shared && aligned)
          k_node_giant<T, true, false, true><<<148, 1024, cap * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant, cap, errw, 0, ncsum);
        else if (shared)
          k_node_giant<T, false, false, true><<<148, 1024, cap * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant, cap, errw, 0, ncsum);
        else if (aligned)
          k_node_giant<T, true><<<148, 1024, cap * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant, cap, errw, 0, ncsum);
        else
          k_node_giant<T, false><<<148, 1024, cap * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant, cap, errw, 0, ncsum);
      }));
      // ---- a5 (nodes): exclusive scan of the per-chunk list totals -> chunk bases, nnz; the node
      // offsets are written by k_node_compact_cb (block scan of the counts + the chunk base) ----
      const int64_t nch_nodes = tiles_of(P.N, kNodeThreads);
      if (P.N > 0) {   // N == 0 with M > 0 always fails validation; nothing to scan
        MN_CUDA(launch("scan_counts", 12.0 * nch_nodes, s, [&] {
          k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch_nodes, kScanTile), kScanThreads, 0, s>>>(
              ncsum, nch_nodes, ncb, sstatus, tickets + 31, 2);
        }));
        MN_CUDA(read_words(host + 1, ncb + nch_nodes, 8, s));
      } else {
        host[1] = 0;
      }
    }
    // ---- a6: the one blocking read (validation word, node nnz) ----
    MN_CUDA(read_words(host, errw, 8, s));
    MN_CUDA(cudaStreamSynchronize(s));
    st = decode_err(host[0], err);
    if (st != MN_OK) goto done;
    if (want_node) {
      U = (int64_t)host[1];
      prof_add_bytes("node_gather", 4.0 * U);
      int32_t* out = U ? (int32_t*)mem.get((size_t)U * 4) : nullptr;
      if (U && !out) { st = MN_ERR_OOM; goto done; }
      if (P.N > 0) {   // (also when nnz == 0: it writes the offsets)
        MN_CUDA(launch("node_compact", 8.0 * U + 24.0 * P.N, s, [&] {
          k_node_compact_cb<<<(unsigned)tiles_of(P.N, kNodeThreads), kNodeThreads, 0, s>>>(eoff, CE, ekA, lofs, cnt,
                                                                                            ncb, P.N, node_off, out);
        }));
      } else {
        MN_CUDA(cudaMemsetAsync(node_off, 0, 8, s));
      }
      node_out->num_nodes = P.N;
      node_out->nnz = U;
      node_out->offsets = node_off;
      node_out->indices = out;
      node_out->owner = mem.a;
    }
    if (want_elem) {
      elem_out->num_nodes = P.N;
      elem_out->nnz = P.Pe;
      elem_out->offsets = elem_off;
      elem_out->indices = elem_idx;
      elem_out->owner = mem.a;
    }
    mem.put(ws);
    return MN_OK;
  }
done:
  if (sink && sink->issued) cudaStreamSynchronize(sink->side);
  if (ws) { cudaStreamSynchronize(s); mem.put(ws); }
  mem.put(node_off);
  mem.put(elem_off);
  mem.put(elem_idx);
  if (want_node && node_out) std::memset(node_out, 0, sizeof(*node_out));
  if (want_elem && elem_out) std::memset(elem_out, 0, sizeof(*elem_out));
  return st;
}

// ================================================================================================
// Memory-bounded mode (the paper's stated shortcoming): the
// nodes are processed in K contiguous ranges, each range by the transpose + expansion path
// restricted to its nodes (the multi-GPU partition applied in time).  The workspace per range is
// ~ (4C + 4) bytes per incidence of the range; element slices land directly in the outputs, node
// slices are concatenated at the end.
// ================================================================================================
static size_t chunk_workspace(const Plan& P, int64_t K) {
  const double inc = (double)P.Pe / (double)K * 1.25 + 64.0;     // incidences of a range (+ imbalance)
  const double nodes = (double)P.N / (double)K + 2.0;
  return (size_t)(4.0 * P.C * inc + 48.0 * nodes + 65536.0);
}

template <int T>
static mn_status chunked_both(const Plan& P, const int32_t* conn, Mem& mem, size_t max_ws, int64_t* chunks,
                              mn_csr* node_out, mn_csr* elem_out, mn_error_detail* err) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  constexpr int C = Elem<T>::C;
  const bool aligned = ((uintptr_t)conn & 15) == 0;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  int64_t K = 1;
  while (K < P.N && chunk_workspace(P, K) > max_ws) K *= 2;
  if (chunks) *chunks = K;
  // the K ranges, processed in ascending order from the back of `todo`; a range whose actual
  // workspace (known after its count pass) exceeds max_ws is split in two, so the bound holds for
  // every range except a single node whose own incidences exceed it (processed alone)
  std::vector<std::pair<int64_t, int64_t>> todo;
  for (int64_t k = K - 1; k >= 0; --k) todo.push_back({P.N * k / K, P.N * (k + 1) / K});
  int64_t ranges = 0;
  int64_t* node_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
  int64_t* elem_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
  int32_t* elem_idx = P.Pe ? (int32_t*)mem.get((size_t)P.Pe * 4 + 16) : nullptr;
  int32_t* node_idx = nullptr;
  std::vector<std::pair<int32_t*, int64_t>> parts;
  void* ws = nullptr;
  uint32_t* temp = nullptr;
  int64_t ebase = 0, nbase = 0;
  if (!node_off || !elem_off || (P.Pe && !elem_idx)) { st = MN_ERR_OOM; goto done; }
  MN_CUDA(cudaMemsetAsync(node_off, 0, (size_t)(P.N + 1) * 8, s));
  MN_CUDA(cudaMemsetAsync(elem_off, 0, (size_t)(P.N + 1) * 8, s));
  while (!todo.empty() && P.M > 0) {
    const int64_t lo = todo.back().first, hi = todo.back().second, nloc = hi - lo;
    todo.pop_back();
    if (nloc == 0) continue;
    Arena ar;
    unsigned long long* errw = ar.take<unsigned long long>(2);
    uint32_t* tickets = ar.take<uint32_t>(8);
    unsigned int* ngiant = ar.take<unsigned int>(1);
    unsigned int* nsgiant = ar.take<unsigned int>(1);
    uint64_t* sstatus = ar.take<uint64_t>((size_t)tiles_of(nloc, kScanTile) + 1);
    const int64_t nch = tiles_of(nloc, kChunkNodes);
    int32_t* ecnt = ar.take<int32_t>((size_t)nch + 1);     // per-chunk counts / cursors
    int32_t* cursor = ar.take<int32_t>((size_t)nch + 1);
    const size_t head = ar.off;
    int64_t* cbase = ar.take<int64_t>((size_t)nch + 1);
    int64_t* eoff = ar.take<int64_t>((size_t)nloc + 1);
    int64_t* noff = ar.take<int64_t>((size_t)nloc + 1);
    int32_t* cnt = ar.take<int32_t>((size_t)nloc + 1);
    int32_t* lofs = ar.take<int32_t>((size_t)nloc + 1);
    uint32_t* giants = ar.take<uint32_t>((size_t)nloc + 1);
    uint32_t* sgiants = ar.take<uint32_t>((size_t)nloc + 1);
    ws = mem.get(ar.off);
    if (!ws) { st = MN_ERR_OOM; goto done; }
    {
      char* bb = (char*)ws;
      auto fix = [&](auto* q) { return (decltype(q))(bb + (size_t)q); };
      errw = fix(errw); tickets = fix(tickets); ngiant = fix(ngiant); nsgiant = fix(nsgiant); sstatus = fix(sstatus);
      ecnt = fix(ecnt); cursor = fix(cursor); eoff = fix(eoff); noff = fix(noff); cnt = fix(cnt); lofs = fix(lofs);
      cbase = fix(cbase);
      giants = fix(giants); sgiants = fix(sgiants);
      MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
      MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
      // (1) validation + per-chunk incidence counts of the range, chunk bases
      MN_CUDA(launch("elem_count", 4.0 * P.K * P.M, s, [&] {
        if (aligned) k_chunk_count<T, true, true><<<count_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, ecnt, errw, lo, hi);
        else k_chunk_count<T, false, true><<<count_grid(P.M), 256, 0, s>>>(conn, P.M, P.N, ecnt, errw, lo, hi);
      }));
      MN_CUDA(launch("scan_counts", 12.0 * nch, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch, kScanTile), kScanThreads, 0, s>>>(
            ecnt, nch, cbase, sstatus, tickets, 1);
      }));
      MN_CUDA(read_words(host, errw, 8, s));
      MN_CUDA(read_words(host + 1, cbase + nch, 8, s));
      MN_CUDA(cudaStreamSynchronize(s));
      st = decode_err(host[0], err);
      if (st != MN_OK) goto done;
      const int64_t Ie = (int64_t)host[1];
      if (ar.off + (size_t)C * (size_t)Ie * 4 > max_ws && nloc > 1) {   // over budget: split the range
        mem.put(ws);
        ws = nullptr;
        const int64_t mid = lo + nloc / 2;
        todo.push_back({mid, hi});
        todo.push_back({lo, mid});
        continue;
      }
      ++ranges;
      int32_t* eslice = elem_idx + ebase;
      // (2) element slice: scatter + per-node sort, straight into the output
      temp = Ie ? (uint32_t*)mem.get((size_t)C * Ie * 4) : nullptr;
      if (Ie && !temp) { st = MN_ERR_OOM; goto done; }
      if (Ie) {
        // buckets (element id + local node byte, 5 B per incidence) in the range's node raw region
        int32_t* belem = reinterpret_cast<int32_t*>(temp);
        uint8_t* bnode = reinterpret_cast<uint8_t*>(temp + Ie);
        MN_CUDA(launch("elem_scatter", 4.0 * P.K * P.M + 5.0 * Ie, s, [&] {
          if (aligned)
            k_chunk_scatter<T, true, true><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, cbase, cursor, belem, bnode, errw,
                                                                          lo, hi);
          else
            k_chunk_scatter<T, false, true><<<hist_grid(P.M), 256, 0, s>>>(conn, P.M, cbase, cursor, belem, bnode, errw,
                                                                           lo, hi);
        }));
        MN_CUDA(launch("elem_segsort", 9.0 * Ie + 8.0 * (nloc + 1), s, [&] {
          k_chunk_sort<true><<<(unsigned)nch, kChunkNodes, 0, s>>>(cbase, nloc, belem, bnode, eoff, eslice, sgiants,
                                                                   nsgiant, errw);
        }));
        const int scap = 48 * 1024;
        cudaFuncSetAttribute(k_segsort_giant, cudaFuncAttributeMaxDynamicSharedMemorySize, scap * 4);
        MN_CUDA(launch("segsort_giant", 0.0, s, [&] {
          k_segsort_giant<<<148, 1024, scap * 4, s>>>(eoff, eslice, sgiants, nsgiant, scap, errw);
        }));
        // (3) node slice: per-node expansion + dedupe, counts, offsets
        const RowSrc rs{conn, 0, P.M, nullptr, nullptr, 0};
        const unsigned ng = (unsigned)tiles_of(nloc, kNodeThreads);
        // rows: at least Ie / K distinct elements touch the range (4 K B each); lists added after the sync
        MN_CUDA(launch("node_gather", 8.0 * (nloc + 1) + 4.0 * Ie + 4.0 * Ie + 8.0 * nloc, s, [&] {
          if (aligned)
            k_node_gather_t<T, true><<<ng, kNodeThreads, 0, s>>>(eoff, eslice, rs, nloc, temp, cnt, lofs, giants,
                                                                 ngiant, errw, lo);
          else
            k_node_gather_t<T, false><<<ng, kNodeThreads, 0, s>>>(eoff, eslice, rs, nloc, temp, cnt, lofs, giants,
                                                                  ngiant, errw, lo);
        }));
        const int cap = 48 * 1024;
        cudaFuncSetAttribute(k_node_giant<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
        cudaFuncSetAttribute(k_node_giant<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
        MN_CUDA(launch("node_giant", 0.0, s, [&] {
          if (aligned)
            k_node_giant<T, true><<<148, 1024, cap * 4, s>>>(eoff, eslice, rs, temp, cnt, lofs, giants, ngiant, cap,
                                                            errw, lo);
          else
            k_node_giant<T, false><<<148, 1024, cap * 4, s>>>(eoff, eslice, rs, temp, cnt, lofs, giants, ngiant, cap,
                                                             errw, lo);
        }));
        MN_CUDA(launch("scan_counts", 12.0 * nloc, s, [&] {
          k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nloc, kScanTile), kScanThreads, 0, s>>>(
              cnt, nloc, noff, sstatus, tickets + 1, 2);
        }));
      } else {   // no incidence in the range: both slices empty
        MN_CUDA(cudaMemsetAsync(noff, 0, (size_t)(nloc + 1) * 8, s));
        MN_CUDA(cudaMemsetAsync(eoff, 0, (size_t)(nloc + 1) * 8, s));
      }
      MN_CUDA(launch("shift_offsets", 16.0 * (nloc + 1), s, [&] {
        k_shift_offsets<<<stream_grid(nloc + 1), 256, 0, s>>>(eoff, nloc + 1, ebase, elem_off + lo);
      }));
      MN_CUDA(read_words(host + 1, noff + nloc, 8, s));
      MN_CUDA(cudaStreamSynchronize(s));
      const int64_t U = (int64_t)host[1];
      prof_add_bytes("node_gather", 4.0 * U);
      if (U) {
        int32_t* part = (int32_t*)mem.get((size_t)U * 4);
        if (!part) { st = MN_ERR_OOM; goto done; }
        parts.push_back({part, U});
        MN_CUDA(launch("node_compact", 8.0 * U + 24.0 * nloc, s, [&] {
          k_node_compact<<<(unsigned)tiles_of(nloc, kNodeThreads), kNodeThreads, 0, s>>>(eoff, C, temp, lofs, noff,
                                                                                       nloc, part);
        }));
      }
      MN_CUDA(launch("shift_offsets", 16.0 * (nloc + 1), s, [&] {
        k_shift_offsets<<<stream_grid(nloc + 1), 256, 0, s>>>(noff, nloc + 1, nbase, node_off + lo);
      }));
      ebase += Ie;
      nbase += U;
    }
    mem.put(temp);
    temp = nullptr;
    mem.put(ws);
    ws = nullptr;
  }
  // concatenate the node slices (peak: slices + output = 2 x node nnz)
  if (nbase) {
    node_idx = (int32_t*)mem.get((size_t)nbase * 4);
    if (!node_idx) { st = MN_ERR_OOM; goto done; }
    int64_t o = 0;
    for (auto& pr : parts) {
      MN_CUDA(cudaMemcpyAsync(node_idx + o, pr.first, (size_t)pr.second * 4, cudaMemcpyDeviceToDevice, s));
      o += pr.second;
    }
  }
  for (auto& pr : parts) mem.put(pr.first);
  parts.clear();
  MN_CUDA(cudaStreamSynchronize(s));
  if (chunks) *chunks = std::max<int64_t>(ranges, 1);
  node_out->num_nodes = P.N; node_out->nnz = nbase; node_out->offsets = node_off; node_out->indices = node_idx;
  node_out->owner = mem.a;
  elem_out->num_nodes = P.N; elem_out->nnz = P.Pe; elem_out->offsets = elem_off; elem_out->indices = elem_idx;
  elem_out->owner = mem.a;
  return MN_OK;
done:
  cudaStreamSynchronize(s);
  mem.put(temp);
  mem.put(ws);
  for (auto& pr : parts) mem.put(pr.first);
  mem.put(node_off); mem.put(elem_off); mem.put(elem_idx); mem.put(node_idx);
  std::memset(node_out, 0, sizeof(*node_out));
  std::memset(elem_out, 0, sizeof(*elem_out));
  return st;
}

template <int T>
static mn_status dispatch_key(const Plan& P, const int32_t* conn, Mem& mem, bool wn, bool we,
                              mn_csr* no, mn_csr* eo, mn_error_detail* err) {
  if (P.key64) {
    if (P.bins == 256) return pipeline<T, uint64_t, 256>(P, conn, mem, wn, we, no, eo, err);
    return pipeline<T, uint64_t, 512>(P, conn, mem, wn, we, no, eo, err);
  }
  if (P.bins == 256) return pipeline<T, uint32_t, 256>(P, conn, mem, wn, we, no, eo, err);
  return pipeline<T, uint32_t, 512>(P, conn, mem, wn, we, no, eo, err);
}

static mn_status check_args(int t, const void* conn, int64_t M, int64_t N) {
  if (t < 0 || t > 3 || M < 0 || N < 0 || N > INT32_MAX) return MN_ERR_INVALID_ARG;
  if (M > 0 && !conn) return MN_ERR_INVALID_ARG;
  if (M > INT32_MAX) return MN_ERR_CAPACITY;   // element ids are int32 in the output
  return MN_OK;
}

// The one-CTA path (small.cuh).  *fallback = true (and nothing returned) when a node's lists are
// too long for it; the caller then runs the staged path.
template <int T>
static mn_status small_path(const Plan& P, const int32_t* conn, Mem& mem, bool wn, bool we, mn_csr* no,
                            mn_csr* eo, mn_error_detail* err, bool* fallback) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  *fallback = false;
  uint64_t* host = pinned_pair();   // the kernel writes (error, nnz, fallback) here directly
  if (!host) return MN_ERR_CUDA;
  const bool aligned = ((uintptr_t)conn & 15) == 0;
  const size_t smem = small_smem_bytes(P.N, P.Pe, P.C);
  static PerDevice attr;
  attr.once([&] {
    const int mx = (int)small_smem_bytes(kSmallMaxN, kSmallMaxPe, 3);
    cudaFuncSetAttribute(k_small_both<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_small_both<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    return 0;
  });
  int64_t *node_off = nullptr, *elem_off = nullptr;
  int32_t *elem_idx = nullptr, *node_idx = nullptr;
  // node indices: one allocation of capacity C * Pe (<= 96 KB), filled in node order, nnz <= capacity
  if (wn) {
    node_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
    node_idx = (int32_t*)mem.get((size_t)P.C * P.Pe * 4);
  }
  if (we) {
    elem_off = (int64_t*)mem.get((size_t)(P.N + 1) * 8);
    elem_idx = (int32_t*)mem.get((size_t)P.Pe * 4 + 16);
  }
  if ((wn && (!node_off || !node_idx)) || (we && (!elem_off || !elem_idx))) { st = MN_ERR_OOM; goto done; }
  MN_CUDA(launch("small_both", 4.0 * P.K * P.M + 8.0 * (P.N + 1) * ((wn ? 1 : 0) + (we ? 1 : 0)) +
                                   (we ? 4.0 * P.Pe : 0.0), s, [&] {
    if (aligned)
      k_small_both<T, true><<<1, kSmallThreads, smem, s>>>(conn, (int)P.M, (int)P.N, elem_off, elem_idx, node_off,
                                                            (uint32_t*)node_idx, (unsigned long long*)host);
    else
      k_small_both<T, false><<<1, kSmallThreads, smem, s>>>(conn, (int)P.M, (int)P.N, elem_off, elem_idx, node_off,
                                                             (uint32_t*)node_idx, (unsigned long long*)host);
  }));
  MN_CUDA(cudaStreamSynchronize(s));
  st = decode_err(host[0], err);
  if (st != MN_OK) goto done;
  if (host[2]) { *fallback = true; goto done; }
  if (wn) {
    const int64_t U = (int64_t)host[1];
    prof_add_bytes("small_both", 4.0 * U);
    no->num_nodes = P.N; no->nnz = U; no->offsets = node_off; no->indices = node_idx; no->owner = mem.a;
  }
  if (we) {
    eo->num_nodes = P.N; eo->nnz = P.Pe; eo->offsets = elem_off; eo->indices = elem_idx; eo->owner = mem.a;
  }
  return MN_OK;
done:
  cudaStreamSynchronize(s);
  mem.put(node_off); mem.put(elem_off); mem.put(elem_idx); mem.put(node_idx);
  if (wn && no) std::memset(no, 0, sizeof(*no));
  if (we && eo) std::memset(eo, 0, sizeof(*eo));
  return st;
}

template <int T>
static mn_status dispatch_inc(const Plan& P, const int32_t* conn, Mem& mem, bool wn, bool we, mn_csr* no,
                              mn_csr* eo, mn_error_detail* err, HostSink* sink, bool shared) {
  if (!sink && !shared && g_elem_path.load() == 0 && P.M > 0 && P.Pe <= g_small_max.load() && P.N <= kSmallMaxN &&
      small_smem_bytes(P.N, P.Pe, P.C) <= small_smem_bytes(kSmallMaxN, kSmallMaxPe, 3)) {
    bool fallback = false;
    const mn_status st = small_path<T>(P, conn, mem, wn, we, no, eo, err, &fallback);
    if (!fallback) return st;
  }
  if (P.bins == 256) return pipeline_inc<T, 256>(P, conn, mem, wn, we, no, eo, err, sink, shared);
  return pipeline_inc<T, 512>(P, conn, mem, wn, we, no, eo, err, sink, shared);
}

// sortpairs = the paper's node pipeline verbatim (node pairs -> global LSD sort -> unique);
// otherwise the element-CSR expansion path (identical output).
static mn_status find(int t, const int32_t* conn, int64_t M, int64_t N, const mn_allocator* a,
                      mn_stream stream, bool wn, bool we, mn_csr* no, mn_csr* eo, mn_error_detail* err,
                      bool sortpairs = false, HostSink* sink = nullptr, bool shared = false) {
  const NvtxScope range(sortpairs ? "mn_find_node_neighbors_sortpairs" : shared ? "mn_find_node_neighbors_shared"
                        : (wn && we) ? "mn_find_neighbors_both" : wn ? "mn_find_node_neighbors"
                        : "mn_find_elem_neighbors");
  if (err) { err->elem = -1; err->pos = -1; }
  mn_status st = check_args(t, conn, M, N);
  if (st != MN_OK) return st;
  if ((wn && !no) || (we && !eo)) return MN_ERR_INVALID_ARG;
  Mem mem(a, (cudaStream_t)stream);
  const Plan P = make_plan(t, M, N);
  if (sortpairs) {
    switch (t) {
      case MN_TRI3: return dispatch_key<MN_TRI3>(P, conn, mem, wn, we, no, eo, err);
      case MN_QUAD4: return dispatch_key<MN_QUAD4>(P, conn, mem, wn, we, no, eo, err);
      case MN_TET4: return dispatch_key<MN_TET4>(P, conn, mem, wn, we, no, eo, err);
      default: return dispatch_key<MN_HEX8>(P, conn, mem, wn, we, no, eo, err);
    }
  }
  switch (t) {
    case MN_TRI3: return dispatch_inc<MN_TRI3>(P, conn, mem, wn, we, no, eo, err, sink, shared);
    case MN_QUAD4: return dispatch_inc<MN_QUAD4>(P, conn, mem, wn, we, no, eo, err, sink, shared);
    case MN_TET4: return dispatch_inc<MN_TET4>(P, conn, mem, wn, we, no, eo, err, sink, shared);
    default: return dispatch_inc<MN_HEX8>(P, conn, mem, wn, we, no, eo, err, sink, shared);
  }
}

// ================================================================================================
// Polygon / mixed-arity surface meshes (kernels in poly.cuh).  Transpose
// path with variable-length rings; outputs any of: ring-edge node CSR, element CSR, element-sharing
// node CSR.  Three blocking reads: the offset bounds, validation + offsets (also sizes the raw
// regions), and the node nnz values.
// ================================================================================================
static mn_status decode_poly_err(uint64_t w, mn_error_detail* err) {
  if (w == ERR_NONE) return MN_OK;
  const int kind = (int)((w >> 22) & 3);
  if (err) {
    err->elem = (int64_t)(w >> 24);
    err->pos = kind >= 2 ? -1 : (int32_t)(w & 0x3FFFFF);
  }
  switch (kind) {
    case 0: return MN_ERR_INDEX_OUT_OF_RANGE;
    case 1: return MN_ERR_DEGENERATE;
    case 2: return MN_ERR_ARITY;
    default: return MN_ERR_INVALID_ARG;
  }
}

static mn_status poly_find(const int64_t* off, const int32_t* idx, int64_t M, int64_t L, int64_t N, Mem& mem,
                           mn_csr* node_out, mn_csr* elem_out, mn_csr* shared_out, mn_error_detail* err) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  const bool wn = node_out != nullptr, we = elem_out != nullptr, wsh = shared_out != nullptr;
  const int64_t scan_tiles = tiles_of(N, kScanTile);
  const unsigned ng = (unsigned)tiles_of(N, kNodeThreads);
  constexpr int cap = 48 * 1024;   // giant raw entries staged in shared memory
  int64_t *elem_off = nullptr, *node_off = nullptr, *sh_off = nullptr;
  int32_t *elem_idx = nullptr, *nidx = nullptr, *sidx = nullptr;
  uint32_t *tempR = nullptr, *tempS = nullptr;
  void* ws = nullptr;
  int64_t rawtotal = 0, Un = 0, Us = 0;
  // workspace pieces
  unsigned long long* errw = nullptr;
  uint32_t *tickets = nullptr, *giants = nullptr, *sgiants = nullptr;
  unsigned int *ngiant = nullptr, *nsgiant = nullptr;
  uint64_t* sstatus = nullptr;
  int32_t *cinc = nullptr, *cursor = nullptr, *rawcnt = nullptr, *cntR = nullptr, *lofsR = nullptr,
          *cntS = nullptr, *lofsS = nullptr;
  int64_t *eoff = nullptr, *rawoff = nullptr;
  int32_t* eidx = nullptr;
  size_t head = 0;
  // node / element outputs of a non-empty mesh: chunk-bucketed transpose (single read of the rings
  // into fixed-capacity 128-node chunk buckets, guarded counted fallback; kernels.cuh / poly.cuh).
  // The element-sharing adjacency needs per-node raw candidate counts: the counted per-node path.
  const bool chunk = !wsh && M > 0 && N > 0;
  const int64_t nch = tiles_of(N, kChunkNodes);
  int32_t* ccur = nullptr;
  unsigned int* ovf = nullptr;
  int64_t* cbase = nullptr;
  uint8_t* bnode = nullptr;
  int ccap = 0;
  auto fill = [&](mn_csr* o, int64_t* offs, int32_t* ind, int64_t nnz) {
    o->num_nodes = N; o->nnz = nnz; o->offsets = offs; o->indices = ind; o->owner = mem.a;
  };
  // the offsets must span exactly [0, conn_len] (an argument error, reported before any element's)
  if (read_words(host, off, 8, s) != cudaSuccess ||
      read_words(host + 1, off + M, 8, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return MN_ERR_CUDA;
  if ((int64_t)host[0] != 0 || (int64_t)host[1] != L) return MN_ERR_INVALID_ARG;
  if (wn) { node_off = (int64_t*)mem.get((size_t)(N + 1) * 8); if (!node_off) { st = MN_ERR_OOM; goto done; } }
  if (wsh) { sh_off = (int64_t*)mem.get((size_t)(N + 1) * 8); if (!sh_off) { st = MN_ERR_OOM; goto done; } }
  if (we) {
    elem_off = (int64_t*)mem.get((size_t)(N + 1) * 8);
    elem_idx = L ? (int32_t*)mem.get((size_t)L * 4) : nullptr;
    if (!elem_off || (L && !elem_idx)) { st = MN_ERR_OOM; goto done; }
  }
  {
    auto layout = [&](Arena& a) {
      errw = a.take<unsigned long long>(2);
      tickets = a.take<uint32_t>(32);
      ngiant = a.take<unsigned int>(1);
      nsgiant = a.take<unsigned int>(1);
      sstatus = a.take<uint64_t>((size_t)scan_tiles + 1);
      cinc = a.take<int32_t>((size_t)N + 1);
      cursor = a.take<int32_t>((size_t)N + 1);
      if (wsh) rawcnt = a.take<int32_t>((size_t)N + 1);
      if (chunk) { ccur = a.take<int32_t>((size_t)nch + 1); ovf = a.take<unsigned int>(1); }
      head = a.off;
      if (chunk) { cbase = a.take<int64_t>((size_t)nch + 1); bnode = a.take<uint8_t>((size_t)2 * L); }
      sgiants = a.take<uint32_t>((size_t)N + 1);
      giants = a.take<uint32_t>((size_t)N + 1);
      eoff = we ? elem_off : a.take<int64_t>((size_t)N + 1);
      eidx = we ? elem_idx : a.take<int32_t>((size_t)L);
      if (wsh) rawoff = a.take<int64_t>((size_t)N + 1);
      if (wn) { cntR = a.take<int32_t>((size_t)N + 1); lofsR = a.take<int32_t>((size_t)N + 1); }
      if (wsh) { cntS = a.take<int32_t>((size_t)N + 1); lofsS = a.take<int32_t>((size_t)N + 1); }
    };
    Arena ar;
    layout(ar);
    ws = mem.get(ar.off);
    if (!ws) { st = MN_ERR_OOM; goto done; }
    ar = Arena{};
    ar.base = (char*)ws;
    layout(ar);
  }
  MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
  MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
  if (chunk) {
    // buckets: element ids in tempR (2 L entries; the ring-edge gather's raw region afterwards),
    // local node bytes in bnode; capacity twice the mean chunk load
    tempR = (uint32_t*)mem.get((size_t)2 * L * 4 + 16);
    if (!tempR) { st = MN_ERR_OOM; goto done; }
    int32_t* belem = reinterpret_cast<int32_t*>(tempR);
    int64_t capl = (2 * L / nch) & ~(int64_t)31;
    const int ovr = g_chunk_cap.load();
    if (ovr > 0 && ovr < capl) capl = ovr;
    if (capl > (int64_t)INT32_MAX - 4096) capl = (int64_t)INT32_MAX - 4096;
    ccap = (int)capl;
    MN_CUDA(launch("poly_scatter", 16.0 * M + 9.0 * L, s, [&] {
      k_poly_chunk_scatter<true><<<hist_grid(M), 256, 0, s>>>(off, idx, M, L, N, ccap, nullptr, ccur, belem, bnode,
                                                              errw, ovf);
    }));
    MN_CUDA(launch("scan_counts", 12.0 * nch, s, [&] {
      k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch, kScanTile), kScanThreads, 0, s>>>(
          ccur, nch, cbase, sstatus, tickets + 29, 1);
    }));
    MN_CUDA(launch("count_fallback", 0.0, s, [&] {
      k_poly_chunk_count<<<hist_grid(M), 256, 0, s>>>(off, idx, M, cinc, errw, ovf);
    }));
    MN_CUDA(launch("scan_fallback", 0.0, s, [&] {
      k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch, kScanTile), kScanThreads, 0, s>>>(
          cinc, nch, cbase, sstatus, tickets + 28, 3, ovf);
    }));
    MN_CUDA(launch("scatter_fallback", 0.0, s, [&] {
      k_poly_chunk_scatter<false><<<hist_grid(M), 256, 0, s>>>(off, idx, M, L, N, 0, cbase, cursor, belem, bnode,
                                                               errw, ovf);
    }));
    MN_CUDA(launch("elem_segsort", 9.0 * L + 8.0 * (N + 1), s, [&] {
      // element lists sorted (R3), also for node-only calls (ascending row visits in the gather)
      k_chunk_sort<true><<<(unsigned)nch, kChunkNodes, 0, s>>>(cbase, N, belem, bnode, eoff, eidx, sgiants,
                                                                nsgiant, errw, ovf, ccap);
    }));
  } else if (M == 0) {
    MN_CUDA(cudaMemsetAsync(eoff, 0, (size_t)(N + 1) * 8, s));
  } else {
    MN_CUDA(launch("poly_count", 16.0 * M + 4.0 * L, s, [&] {
      k_poly_count<<<hist_grid(M), 256, 0, s>>>(off, idx, M, L, N, cinc, wsh ? rawcnt : nullptr, errw);
    }));
    if (N > 0) {
      MN_CUDA(launch("scan_counts", 12.0 * N, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)scan_tiles, kScanThreads, 0, s>>>(cinc, N, eoff, sstatus,
                                                                                 tickets + 29, 1);
      }));
      if (wsh)
        MN_CUDA(launch("scan_counts", 12.0 * N, s, [&] {
          k_scan_i32<kScanThreads, kScanItems><<<(unsigned)scan_tiles, kScanThreads, 0, s>>>(rawcnt, N, rawoff, sstatus,
                                                                                   tickets + 28, 3);
        }));
    }
  }
  // ---- blocking read 1: validation word (+ the element-sharing raw total) ----
  MN_CUDA(read_words(host, errw, 8, s));
  if (wsh && M > 0 && N > 0) MN_CUDA(read_words(host + 1, rawoff + N, 8, s));
  MN_CUDA(cudaStreamSynchronize(s));
  st = decode_poly_err(host[0], err);
  if (st != MN_OK) goto done;
  rawtotal = (wsh && M > 0 && N > 0) ? (int64_t)host[1] : 0;
  if (M > 0) {
    if (!chunk)
      MN_CUDA(launch("poly_scatter", 16.0 * M + 16.0 * L, s, [&] {
        k_poly_scatter<<<hist_grid(M), 256, 0, s>>>(off, idx, M, eoff, cursor, eidx, errw);
      }));
    if (we) {
      if (!chunk)
        MN_CUDA(launch("elem_segsort", 8.0 * L + 8.0 * (N + 1), s, [&] {
          segsort_fn<<<(unsigned)tiles_of(N, kSegThreads), kSegThreads, 0, s>>>(eoff, N, eidx, sgiants, nsgiant,
                                                                                   errw);
        }));
      static PerDevice seg_attr;
      seg_attr.once([&] {
        cudaFuncSetAttribute(k_segsort_giant, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
        return 0;
      });
      MN_CUDA(launch("segsort_giant", 0.0, s, [&] {
        k_segsort_giant<<<148, 1024, cap * 4, s>>>(eoff, eidx, sgiants, nsgiant, cap, errw);
      }));
    }
    static PerDevice poly_attr;
    poly_attr.once([&] {
      cudaFuncSetAttribute(k_poly_giant<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
      cudaFuncSetAttribute(k_poly_giant<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
      return 0;
    });
    if (wn) {   // ring-edge node adjacency: 2 raw candidates per incidence
      if (!tempR) tempR = L ? (uint32_t*)mem.get((size_t)2 * L * 4) : nullptr;
      if (L && !tempR) { st = MN_ERR_OOM; goto done; }
      // element CSR, every ring once (offsets + entries), counts + list offsets; lists added after the sync
      MN_CUDA(launch("poly_gather", 8.0 * (N + 1) + 4.0 * L + 8.0 * (M + 1) + 4.0 * L + 8.0 * N, s, [&] {
        k_poly_gather<false><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, off, idx, N, nullptr, 2, tempR, cntR, lofsR,
                                                        giants, ngiant, errw);
      }));
      MN_CUDA(launch("poly_giant", 0.0, s, [&] {
        k_poly_giant<false><<<148, 1024, cap * 4, s>>>(eoff, eidx, off, idx, nullptr, 2, tempR, cntR, lofsR, giants,
                                                       ngiant, cap, errw);
      }));
      MN_CUDA(launch("scan_counts", 12.0 * N, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)scan_tiles, kScanThreads, 0, s>>>(cntR, N, node_off, sstatus,
                                                                                 tickets + 31, 2);
      }));
      MN_CUDA(read_words(host + 2, node_off + N, 8, s));
    }
    if (wsh) {   // element-sharing adjacency: k_e - 1 raw candidates per incidence
      tempS = rawtotal ? (uint32_t*)mem.get((size_t)rawtotal * 4) : nullptr;
      if (rawtotal && !tempS) { st = MN_ERR_OOM; goto done; }
      MN_CUDA(cudaMemsetAsync(ngiant, 0, 4, s));
      MN_CUDA(launch("poly_gather", 16.0 * (N + 1) + 4.0 * L + 8.0 * (M + 1) + 4.0 * L + 8.0 * N, s, [&] {
        k_poly_gather<true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, off, idx, N, rawoff, 0, tempS, cntS, lofsS,
                                                       giants, ngiant, errw);
      }));
      MN_CUDA(launch("poly_giant", 0.0, s, [&] {
        k_poly_giant<true><<<148, 1024, cap * 4, s>>>(eoff, eidx, off, idx, rawoff, 0, tempS, cntS, lofsS, giants,
                                                      ngiant, cap, errw);
      }));
      MN_CUDA(launch("scan_counts", 12.0 * N, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)scan_tiles, kScanThreads, 0, s>>>(cntS, N, sh_off, sstatus,
                                                                                 tickets + 30, 4);
      }));
      MN_CUDA(read_words(host + 3, sh_off + N, 8, s));
    }
  } else {
    if (wn) MN_CUDA(cudaMemsetAsync(node_off, 0, (size_t)(N + 1) * 8, s));
    if (wsh) MN_CUDA(cudaMemsetAsync(sh_off, 0, (size_t)(N + 1) * 8, s));
    host[2] = host[3] = 0;
  }
  // ---- blocking read 2: node nnz values ----
  MN_CUDA(cudaStreamSynchronize(s));
  Un = (wn && M > 0) ? (int64_t)host[2] : 0;
  Us = (wsh && M > 0) ? (int64_t)host[3] : 0;
  if (wsh) prof_add_bytes("poly_gather", 4.0 * (double)Us);
  if (wn) prof_add_bytes("poly_gather", 4.0 * (double)Un, wsh ? 1 : 0);
  if (Un) {
    nidx = (int32_t*)mem.get((size_t)Un * 4);
    if (!nidx) { st = MN_ERR_OOM; goto done; }
    MN_CUDA(launch("node_compact", 8.0 * Un + 24.0 * N, s, [&] {
      k_node_compact<<<ng, kNodeThreads, 0, s>>>(eoff, 2, tempR, lofsR, node_off, N, nidx);
    }));
  }
  if (Us) {
    sidx = (int32_t*)mem.get((size_t)Us * 4);
    if (!sidx) { st = MN_ERR_OOM; goto done; }
    MN_CUDA(launch("node_compact", 8.0 * Us + 32.0 * N, s, [&] {
      k_node_compact<<<ng, kNodeThreads, 0, s>>>(eoff, 0, tempS, lofsS, sh_off, N, sidx, rawoff);
    }));
  }
  if (wn) fill(node_out, node_off, nidx, Un);
  if (we) fill(elem_out, elem_off, elem_idx, L);
  if (wsh) fill(shared_out, sh_off, sidx, Us);
  mem.put(tempR);
  mem.put(tempS);
  mem.put(ws);
  return MN_OK;
done:
  cudaStreamSynchronize(s);
  mem.put(tempR);
  mem.put(tempS);
  mem.put(ws);
  mem.put(node_off);
  mem.put(sh_off);
  mem.put(elem_off);
  mem.put(elem_idx);
  mem.put(nidx);
  mem.put(sidx);
  for (mn_csr* o : {node_out, elem_out, shared_out})
    if (o) std::memset(o, 0, sizeof(*o));
  return st;
}

// ================================================================================================
// generic LSD sorts (stage entry points and the multi-GPU finish)
// ================================================================================================
template <typename KeyT, bool PAYLOAD>
static mn_status lsd_sort(KeyT* keys, uint32_t* vals, int64_t n, int bits, Mem& mem) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  if (n <= 1 || bits <= 0) return MN_OK;
  const int p = (bits + 7) / 8;
  const int64_t tiles = tiles_of(n, kTile);
  Arena ar;
  unsigned long long* errw = ar.take<unsigned long long>(1);
  uint32_t* tickets = ar.take<uint32_t>(32);
  unsigned long long* hist = ar.take<unsigned long long>((size_t)p * 256);
  uint64_t* bases = ar.take<uint64_t>((size_t)p * 256);
  uint64_t* status = ar.take<uint64_t>((size_t)tiles * 256);
  const size_t head = ar.off;
  KeyT* alt = ar.take<KeyT>(n);
  uint32_t* valt = PAYLOAD ? ar.take<uint32_t>(n) : nullptr;
  void* ws = mem.get(ar.off);
  if (!ws) return MN_ERR_OOM;
  {
    char* b = (char*)ws;
    auto fix = [&](auto* q) { return (decltype(q))(b + (size_t)q); };
    errw = fix(errw); tickets = fix(tickets); hist = fix(hist); bases = fix(bases);
    status = fix(status); alt = fix(alt);
    if (PAYLOAD) valt = fix(valt);
    MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
    MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
    MN_CUDA(launch("hist_keys", (double)sizeof(KeyT) * n, s, [&] {
      k_hist_keys<KeyT><<<stream_grid(n), 256, 0, s>>>(keys, n, p, hist);
    }));
    BasesDesc bd{};
    bd.npass = p;
    for (int q = 0; q < p; ++q) { bd.hidx[q] = q; bd.mult[q] = 1; }
    MN_CUDA(launch("bucket_bases", 0.0, s, [&] { k_bucket_bases<256><<<p, 256, 0, s>>>(hist, bd, bases, errw); }));
    KeyT* kb[2] = {keys, alt};
    uint32_t* vb[2] = {vals, valt};
    for (int q = 0; q < p; ++q) {
      PassArgs pa{};
      pa.keys_in = kb[q & 1];
      pa.keys_out = kb[(q + 1) & 1];
      pa.vals_in = vb[q & 1];
      pa.vals_out = vb[(q + 1) & 1];
      pa.n = n;
      const int width = std::min(8, bits - 8 * q);
      pa.pd = mask_digit(8 * q, width);
      pa.bases = bases + (size_t)q * 256;
      pa.status = status;
      pa.ticket = tickets + q;
      pa.epoch = (uint32_t)(q + 1);
      pa.err = errw;
      MN_CUDA((run_pass<KeyT, 0, 0, PAYLOAD, false, 256>(pa, s, "onesweep_generic",
                                                          (double)(PAYLOAD ? 2 * (sizeof(KeyT) + 4) : 2 * sizeof(KeyT)) * n)));
    }
    if (p & 1) {
      MN_CUDA(cudaMemcpyAsync(keys, alt, (size_t)n * sizeof(KeyT), cudaMemcpyDeviceToDevice, s));
      if (PAYLOAD) MN_CUDA(cudaMemcpyAsync(vals, valt, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
    }
  }
done:
  mem.put(ws);
  return st;
}

// Unique + offsets on arbitrary sorted node keys (stage entry point, multi-GPU finish).
template <typename KeyT>
static mn_status unique_csr(const KeyT* keys, int64_t n, int b, int64_t N, int64_t* offsets,
                            int32_t* indices, int64_t* h_nnz, Mem& mem) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  if (n == 0) {
    if (cudaMemsetAsync(offsets, 0, (size_t)(N + 1) * 8, s) != cudaSuccess) return MN_ERR_CUDA;
    *h_nnz = 0;
    return MN_OK;
  }
  const int64_t tiles = tiles_of(n, kUTile);
  Arena ar;
  unsigned long long* errw = ar.take<unsigned long long>(2);
  uint32_t* ticket = ar.take<uint32_t>(1);
  uint64_t* status = ar.take<uint64_t>((size_t)tiles);
  void* ws = mem.get(ar.off);
  if (!ws) return MN_ERR_OOM;
  {
    char* bb = (char*)ws;
    errw = (unsigned long long*)(bb + (size_t)errw);
    unsigned long long* nnz = errw + 1;
    ticket = (uint32_t*)(bb + (size_t)ticket);
    status = (uint64_t*)(bb + (size_t)status);
    MN_CUDA(cudaMemsetAsync(ws, 0, ar.off, s));
    MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
    UniqueArgs ua{};
    ua.keys = keys; ua.n = n; ua.b = b; ua.N = N; ua.offsets = offsets;
    ua.indices = reinterpret_cast<uint32_t*>(indices);
    ua.status = status; ua.ticket = ticket; ua.epoch = 1; ua.nnz = nnz; ua.err = errw;
    MN_CUDA(launch("unique_node", (double)sizeof(KeyT) * n + 8.0 * (N + 1), s, [&] {
      k_unique_node<KeyT, kThreads, kItems><<<(unsigned)tiles, kThreads, 0, s>>>(ua);
    }));
    MN_CUDA(read_words(host, errw, 16, s));
    MN_CUDA(cudaStreamSynchronize(s));
    *h_nnz = (int64_t)host[1];
  }
done:
  mem.put(ws);
  return st;
}

// Validation + emission kernels for the stage entry points.
template <int T>
static mn_status emit_stage(const int32_t* conn, int64_t M, int64_t N, void* keys, uint32_t* ekeys,
                            uint32_t* evals, bool node, Mem& mem, mn_error_detail* err) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  const Plan P = make_plan(T, M, N);
  Arena ar;
  unsigned long long* errw = ar.take<unsigned long long>(1);
  unsigned long long* hist = ar.take<unsigned long long>(4 * 512);
  void* ws = mem.get(ar.off);
  if (!ws) return MN_ERR_OOM;
  errw = (unsigned long long*)((char*)ws + (size_t)errw);
  hist = (unsigned long long*)((char*)ws + (size_t)hist);
  MN_CUDA(cudaMemsetAsync(ws, 0, ar.off, s));
  MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
  if (M > 0) {
    MN_CUDA(launch("hist_validate", 4.0 * P.K * M, s, [&] {
      k_hist_validate<T, 512, false><<<hist_grid(M), 256, 0, s>>>(conn, M, N, 0, P.dp, 0, 1, hist, errw);
    }));
    if (node) {
      if (P.key64) {
        MN_CUDA(launch("emit_node", 4.0 * P.K * M + 8.0 * P.Pn, s, [&] {
          k_emit_node<T, uint64_t><<<stream_grid(P.Pn), 256, 0, s>>>(conn, P.Pn, P.b, (uint64_t*)keys, errw);
        }));
      } else {
        MN_CUDA(launch("emit_node", 4.0 * P.K * M + 4.0 * P.Pn, s, [&] {
          k_emit_node<T, uint32_t><<<stream_grid(P.Pn), 256, 0, s>>>(conn, P.Pn, P.b, (uint32_t*)keys, errw);
        }));
      }
    } else {
      MN_CUDA(launch("emit_elem", 12.0 * P.Pe, s, [&] {
        k_emit_elem<T><<<stream_grid(P.Pe), 256, 0, s>>>(conn, P.Pe, ekeys, evals, errw);
      }));
    }
  }
  MN_CUDA(read_words(host, errw, 8, s));
  MN_CUDA(cudaStreamSynchronize(s));
  st = decode_err(host[0], err);
done:
  mem.put(ws);
  return st;
}

// ================================================================================================
// multi-GPU bucketing: stable owner partition fused with pair creation (one onesweep pass each)
// ================================================================================================
template <int T, int BINS>
static mn_status dist_bucket_impl(const int32_t* conn, int64_t M, int64_t base, int64_t N, int world, int self,
                                  uint64_t* pairs, int64_t* hc, int32_t** relems_out, int32_t** rrows_out,
                                  int64_t* hrc, Mem& mem, mn_error_detail* err, uint64_t* defer = nullptr) {
  // defer != nullptr (mn_find_neighbors_dist): a validation failure is not returned but stored in
  // *defer (the raw error word, ERR_NONE if none) with all counts 0, so this rank still joins the
  // count exchange, where the lowest word over all ranks decides (every rank returns it)
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  const Plan P = make_plan(T, M, N);
  const uint64_t chunk = (uint64_t)((N + world - 1) / world > 0 ? (N + world - 1) / world : 1);
  const int64_t tiles = tiles_of(P.Pe, kTile);
  std::vector<unsigned long long> hh(BINS), hr(BINS);
  int32_t *relems = nullptr, *rrows = nullptr;
  int64_t R = 0;
  Arena ar;
  unsigned long long* errw = ar.take<unsigned long long>(2);
  uint32_t* tickets = ar.take<uint32_t>(8);
  unsigned long long* hist = ar.take<unsigned long long>(BINS);
  unsigned long long* rcnt = ar.take<unsigned long long>(BINS);
  uint64_t* bases = ar.take<uint64_t>(BINS);
  uint64_t* status = ar.take<uint64_t>((size_t)(tiles ? tiles : 1) * BINS);
  uint64_t* sstatus = ar.take<uint64_t>((size_t)tiles_of(P.Pe, kScanTile) + 1);
  const size_t head = ar.off;
  int32_t* flags = ar.take<int32_t>((size_t)P.Pe + 1);
  int64_t* pos = ar.take<int64_t>((size_t)P.Pe + 1);
  void* ws = mem.get(ar.off);
  if (!ws) return MN_ERR_OOM;
  {
    char* bb = (char*)ws;
    auto fix = [&](auto* q) { return (decltype(q))(bb + (size_t)q); };
    errw = fix(errw); tickets = fix(tickets); hist = fix(hist); rcnt = fix(rcnt); bases = fix(bases);
    status = fix(status); sstatus = fix(sstatus); flags = fix(flags); pos = fix(pos);
    MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
    MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
    if (M > 0) {
      // validation + incidence counts per owner rank
      MN_CUDA(launch("hist_validate", 4.0 * P.K * M, s, [&] {
        k_hist_validate<T, BINS, false><<<hist_grid(M), 256, 0, s>>>(conn, M, N, base, P.dp, 1, chunk, hist, errw);
      }));
      BasesDesc bd{};
      bd.npass = 1;
      bd.hidx[0] = 0;
      bd.mult[0] = 1;
      MN_CUDA(launch("bucket_bases", 0.0, s, [&] { k_bucket_bases<BINS><<<1, BINS, 0, s>>>(hist, bd, bases, errw); }));
      // (node << 32 | global element) pairs created from conn, stably bucketed by owner
      PassArgs pe{};
      pe.keys_out = pairs; pe.conn = conn; pe.elem_base = base; pe.n = P.Pe;
      pe.pd.shift = 32; pe.pd.div = chunk; pe.pd.mask = 0;
      pe.bases = bases; pe.status = status; pe.ticket = tickets; pe.epoch = 1; pe.err = errw;
      MN_CUDA((run_pass<uint64_t, 3, T, false, true, BINS>(pe, s, "bucket_incidences", 4.0 * P.Pe + 8.0 * P.Pe)));
      // one row per (remote destination, element): the owner reads local rows from its own shard
      MN_CUDA(launch("mark_remote_rows", 16.0 * P.Pe, s, [&] {
        k_mark_remote_rows<<<stream_grid(P.Pe), 256, 0, s>>>(pairs, P.Pe, chunk, world, self, flags, errw);
      }));
      MN_CUDA(launch("scan_counts", 12.0 * P.Pe, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(P.Pe, kScanTile), kScanThreads, 0, s>>>(
            flags, P.Pe, pos, sstatus, tickets + 1, 1);
      }));
      MN_CUDA(launch("row_counts", 0.0, s, [&] { k_row_counts<<<1, 512, 0, s>>>(pos, bases, world, P.Pe, rcnt); }));
      MN_CUDA(read_words(host + 1, pos + P.Pe, 8, s));
    }
    MN_CUDA(cudaMemcpyAsync(hh.data(), hist, BINS * 8, cudaMemcpyDeviceToHost, s));
    MN_CUDA(cudaMemcpyAsync(hr.data(), rcnt, BINS * 8, cudaMemcpyDeviceToHost, s));
    MN_CUDA(read_words(host, errw, 8, s));
    MN_CUDA(cudaStreamSynchronize(s));
    if (defer) {
      *defer = host[0];
      if (host[0] != ERR_NONE) {
        for (int g = 0; g < world; ++g) hc[g] = hrc[g] = 0;
        *relems_out = *rrows_out = nullptr;
        goto done;
      }
    }
    st = decode_err(host[0], err);
    if (st != MN_OK) goto done;
    R = M > 0 ? (int64_t)host[1] : 0;
    for (int g = 0; g < world; ++g) {
      hc[g] = (int64_t)hh[g];
      hrc[g] = (int64_t)hr[g];
    }
    if (R > 0) {
      relems = (int32_t*)mem.get((size_t)R * 4);
      rrows = (int32_t*)mem.get((size_t)R * P.K * 4);
      if (!relems || !rrows) { st = MN_ERR_OOM; goto done; }
      MN_CUDA(launch("emit_remote_rows", 8.0 * P.Pe + 4.0 * (P.K + 1) * R, s, [&] {
        k_emit_remote_rows<T><<<stream_grid(P.Pe), 256, 0, s>>>(pairs, flags, pos, P.Pe, conn, base, relems, rrows,
                                                               errw);
      }));
    }
    *relems_out = relems;
    *rrows_out = rrows;
    relems = rrows = nullptr;
  }
done:
  mem.put(relems);
  mem.put(rrows);
  mem.put(ws);
  return st;
}

// Owner-side finish: element CSR slice by a stable sort of the received incidences on the local
// node id (source-rank order keeps element ids ascending; the element ids are the sort payload and
// become the indices in place), node CSR slice by the same per-node expansion + dedupe as the
// single-GPU path, rows read from the own shard or, for remote elements, the received row table.
template <int T>
static mn_status dist_finish_impl(const PairSrc& pairs, int64_t n, const int32_t* relems, const int32_t* rrows,
                                  int64_t nr, const int32_t* shard, int64_t shard_base, int64_t shard_m, int64_t N,
                                  int64_t lo, int64_t hi, Mem& mem, mn_csr* node_slice, mn_csr* elem_slice) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  constexpr int K = Elem<T>::K, C = Elem<T>::C;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  const int64_t nloc = hi - lo;
  const int bl = node_bits(nloc);
  std::memset(node_slice, 0, sizeof(*node_slice));
  std::memset(elem_slice, 0, sizeof(*elem_slice));
  int64_t* noff = (int64_t*)mem.get((size_t)(nloc + 1) * 8);
  int64_t* eoff = (int64_t*)mem.get((size_t)(nloc + 1) * 8);
  int32_t* eidx = n ? (int32_t*)mem.get((size_t)n * 4 + 16) : nullptr;   // +16: aligned 16-byte reads
  void* ws = nullptr;
  if (!noff || !eoff || (n && !eidx)) { st = MN_ERR_OOM; goto done; }
  if (n == 0) {
    MN_CUDA(cudaMemsetAsync(noff, 0, (size_t)(nloc + 1) * 8, s));
    MN_CUDA(cudaMemsetAsync(eoff, 0, (size_t)(nloc + 1) * 8, s));
    MN_CUDA(cudaStreamSynchronize(s));
  } else {
    Arena ar;
    unsigned long long* errw = ar.take<unsigned long long>(2);
    unsigned long long* smp = ar.take<unsigned long long>(2);
    uint32_t* tickets = ar.take<uint32_t>(8);
    unsigned int* ngiant = ar.take<unsigned int>(1);
    uint64_t* sstatus = ar.take<uint64_t>((size_t)tiles_of(nloc, kScanTile) + 1);
    int32_t* cnt = ar.take<int32_t>((size_t)nloc + 1);    // zeroed: counts of the transpose
    int32_t* lofs = ar.take<int32_t>((size_t)nloc + 1);   // zeroed: cursors of the transpose
    const int64_t nch = tiles_of(nloc, kChunkNodes);
    int32_t* ccur = ar.take<int32_t>((size_t)nch + 1);     // zeroed: fixed chunk-bucket cursors
    unsigned int* ovf = ar.take<unsigned int>(1);          // zeroed: a fixed bucket overflowed
    const size_t head = ar.off;
    uint32_t* keys = ar.take<uint32_t>((size_t)n);
    uint32_t* temp = ar.take<uint32_t>((size_t)C * n);
    uint32_t* giants = ar.take<uint32_t>((size_t)nloc + 1);
    ws = mem.get(ar.off);
    if (!ws) { st = MN_ERR_OOM; goto done; }
    {
      char* bb = (char*)ws;
      auto fix = [&](auto* q) { return (decltype(q))(bb + (size_t)q); };
      errw = fix(errw); smp = fix(smp); tickets = fix(tickets); ngiant = fix(ngiant); sstatus = fix(sstatus);
      keys = fix(keys); temp = fix(temp); cnt = fix(cnt); lofs = fix(lofs); giants = fix(giants);
      ccur = fix(ccur); ovf = fix(ovf);
      uint32_t* elems = reinterpret_cast<uint32_t*>(eidx);
      MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
      MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
      // element CSR slice: counting-sort transpose when the received pairs have locality (same rule
      // as the 1-GPU path), else a stable LSD sort on the local node id
      bool transpose = g_elem_path.load() == 2;
      if (g_elem_path.load() == 0 && n >= kTransposeMinElems) {
        MN_CUDA(launch("locality_sample", 0.0, s, [&] { k_pairs_locality<<<64, 256, 0, s>>>(pairs, n, smp); }));
        MN_CUDA(read_words(host + 2, smp, 16, s));
        MN_CUDA(cudaStreamSynchronize(s));
        transpose = host[3] > 0 && (double)host[2] < kTransposeMaxGroupRatio * (double)host[3];
      }
      if (transpose) {
        if (nloc > 0) {
          // chunk-bucketed: the pairs into fixed-capacity 128-node chunk buckets (element ids in temp,
          // node bytes in keys; both dead until the node pass), guarded counted fallback, chunk sort
          int32_t* belem = reinterpret_cast<int32_t*>(temp);
          uint8_t* bnode = reinterpret_cast<uint8_t*>(keys);
          int64_t* cbase = noff;   // scratch until the node scan writes the node offsets
          int64_t capl = (2 * n / nch) & ~(int64_t)31;
          const int ovr = g_chunk_cap.load();
          if (ovr > 0 && ovr < capl) capl = ovr;
          if (capl > (int64_t)INT32_MAX - 4096) capl = (int64_t)INT32_MAX - 4096;
          const int cap = (int)capl;
          MN_CUDA(launch("elem_scatter", 8.0 * n + 5.0 * n, s, [&] {
            k_pairs_chunk_scatter<true><<<stream_grid(n), 256, 0, s>>>(pairs, n, lo, cap, nullptr, ccur, belem,
                                                                        bnode, ovf);
          }));
          MN_CUDA(launch("scan_counts", 12.0 * nch, s, [&] {
            k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch, kScanTile), kScanThreads, 0, s>>>(
                ccur, nch, cbase, sstatus, tickets + 2, 1);
          }));
          MN_CUDA(launch("count_fallback", 0.0, s, [&] {
            k_pairs_chunk_count<<<stream_grid(n), 256, 0, s>>>(pairs, n, lo, cnt, ovf);
          }));
          MN_CUDA(launch("scan_fallback", 0.0, s, [&] {
            k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch, kScanTile), kScanThreads, 0, s>>>(
                cnt, nch, cbase, sstatus, tickets + 3, 3, ovf);
          }));
          MN_CUDA(launch("scatter_fallback", 0.0, s, [&] {
            k_pairs_chunk_scatter<false><<<stream_grid(n), 256, 0, s>>>(pairs, n, lo, 0, cbase, lofs, belem, bnode,
                                                                         ovf);
          }));
          MN_CUDA(launch("elem_segsort", 9.0 * n + 8.0 * (nloc + 1), s, [&] {
            k_chunk_sort<true><<<(unsigned)nch, kChunkNodes, 0, s>>>(cbase, nloc, belem, bnode, eoff, eidx, giants,
                                                                      ngiant, errw, ovf, cap);
          }));
          const int scap = 48 * 1024;
          cudaFuncSetAttribute(k_segsort_giant, cudaFuncAttributeMaxDynamicSharedMemorySize, scap * 4);
          MN_CUDA(launch("segsort_giant", 0.0, s, [&] {
            k_segsort_giant<<<148, 1024, scap * 4, s>>>(eoff, eidx, giants, ngiant, scap, errw);
          }));
          // reset the buffers the node pass reuses (counts, cursors, giant queue)
          MN_CUDA(cudaMemsetAsync(cnt, 0, (size_t)(nloc + 1) * 4, s));
          MN_CUDA(cudaMemsetAsync(lofs, 0, (size_t)(nloc + 1) * 4, s));
          MN_CUDA(cudaMemsetAsync(ngiant, 0, 4, s));
        } else {
          MN_CUDA(cudaMemsetAsync(eoff, 0, 8, s));
        }
      } else {
        MN_CUDA(launch("local_keys", 16.0 * n, s, [&] {
          k_local_keys<<<stream_grid(n), 256, 0, s>>>(pairs, n, lo, keys, elems);
        }));
        st = lsd_sort<uint32_t, true>(keys, elems, n, bl, mem);
        if (st != MN_OK) goto done;
        MN_CUDA(launch("elem_offsets", 4.0 * n + 8.0 * (nloc + 1), s, [&] {
          k_elem_offsets<false><<<stream_grid(n / 4 + 1), 256, 0, s>>>(keys, n, nloc, eoff, nullptr);
        }));
      }
      if (nloc > 0) {
        const bool aligned = ((uintptr_t)shard & 15) == 0 && ((uintptr_t)rrows & 15) == 0;
        const RowSrc rs{shard, shard_base, shard_m, relems, rrows, nr};
        const unsigned ng = (unsigned)tiles_of(nloc, kNodeThreads);
        MN_CUDA(launch("node_gather", 8.0 * (nloc + 1) + 4.0 * n + 4.0 * K * n, s, [&] {
          if (aligned)
            k_node_gather_t<T, true, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, nloc, temp, cnt, lofs,
                                                                       giants, ngiant, errw, lo);
          else
            k_node_gather_t<T, false, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, nloc, temp, cnt, lofs,
                                                                        giants, ngiant, errw, lo);
        }));
        const int cap = 48 * 1024;
        static PerDevice attr;
        attr.once([&] {
          cudaFuncSetAttribute(k_node_giant<T, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
          cudaFuncSetAttribute(k_node_giant<T, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
          return 0;
        });
        MN_CUDA(launch("node_giant", 0.0, s, [&] {
          if (aligned)
            k_node_giant<T, true, true><<<148, 1024, cap * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant,
                                                                  cap, errw, lo);
          else
            k_node_giant<T, false, true><<<148, 1024, cap * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant,
                                                                   cap, errw, lo);
        }));
        MN_CUDA(launch("scan_counts", 12.0 * nloc, s, [&] {   // epoch 2: the element scan may have used 1
          k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nloc, kScanTile), kScanThreads, 0, s>>>(
              cnt, nloc, noff, sstatus, tickets + 1, 2);
        }));
      } else {
        MN_CUDA(cudaMemsetAsync(noff, 0, 8, s));
      }
      MN_CUDA(read_words(host + 1, noff + nloc, 8, s));
      MN_CUDA(cudaStreamSynchronize(s));
      const int64_t U = (int64_t)host[1];
      if (U) {
        node_slice->indices = (int32_t*)mem.get((size_t)U * 4);
        if (!node_slice->indices) { st = MN_ERR_OOM; goto done; }
        MN_CUDA(launch("node_compact", 8.0 * U + 24.0 * nloc, s, [&] {
          k_node_compact<<<(unsigned)tiles_of(nloc, kNodeThreads), kNodeThreads, 0, s>>>(
              eoff, C, temp, lofs, noff, nloc, node_slice->indices);
        }));
      }
      node_slice->nnz = U;
    }
  }
  node_slice->num_nodes = nloc;
  node_slice->offsets = noff;
  node_slice->owner = mem.a;
  elem_slice->num_nodes = nloc;
  elem_slice->nnz = n;
  elem_slice->offsets = eoff;
  elem_slice->indices = eidx;
  elem_slice->owner = mem.a;
  mem.put(ws);
  if (cudaStreamSynchronize(s) != cudaSuccess) return MN_ERR_CUDA;
  return MN_OK;
done:
  cudaStreamSynchronize(s);
  mem.put(ws);
  mem.put(noff);
  mem.put(eoff);
  mem.put(eidx);
  if (node_slice->indices) mem.put(node_slice->indices);
  std::memset(node_slice, 0, sizeof(*node_slice));
  std::memset(elem_slice, 0, sizeof(*elem_slice));
  return st;
}

#include "dist.cuh"

}  // namespace mn

// ==================================================================================================
// C ABI
// ==================================================================================================
using namespace mn;

extern "C" {

int mn_abi_version(void) { return MN_ABI_VERSION; }

const char* mn_status_string(mn_status s) {
  switch (s) {
    case MN_OK: return "ok";
    case MN_ERR_INVALID_ARG: return "invalid argument";
    case MN_ERR_INDEX_OUT_OF_RANGE: return "node index out of range";
    case MN_ERR_DEGENERATE: return "degenerate element (repeated node)";
    case MN_ERR_CAPACITY: return "capacity exceeded";
    case MN_ERR_OOM: return "out of device memory";
    case MN_ERR_CUDA: return "CUDA error";
    case MN_ERR_ARITY: return "element with fewer than 3 nodes";
    case MN_ERR_SYNTAX: return "mesh file syntax error";
    case MN_ERR_COUNT_MISMATCH: return "mesh file count mismatch";
    case MN_ERR_ZERO_INDEX: return "OBJ face index 0";
    case MN_ERR_COMM: return "multi-GPU exchange failed (NCCL / mn_comm)";
  }
  return "unknown status";
}

int mn_node_key_bits(int64_t num_nodes) { return node_bits(num_nodes); }
int mn_node_key_bytes(int64_t num_nodes) { return 2 * node_bits(num_nodes) > 32 ? 8 : 4; }

mn_status mn_find_node_neighbors(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N,
                                 const mn_allocator* a, mn_stream s, mn_csr* out, mn_error_detail* err) {
  return find(t, d_conn, M, N, a, s, true, false, out, nullptr, err);
}

mn_status mn_find_node_neighbors_sortpairs(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N,
                                           const mn_allocator* a, mn_stream s, mn_csr* out, mn_error_detail* err) {
  return find(t, d_conn, M, N, a, s, true, false, out, nullptr, err, true);
}

mn_status mn_find_node_neighbors_shared(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N,
                                        const mn_allocator* a, mn_stream s, mn_csr* out, mn_error_detail* err) {
  return find(t, d_conn, M, N, a, s, true, false, out, nullptr, err, false, nullptr, true);
}

mn_status mn_find_poly_neighbors(const int64_t* d_off, const int32_t* d_idx, int64_t num_elems, int64_t conn_len,
                                 int64_t num_nodes, const mn_allocator* a, mn_stream s, mn_csr* node_out,
                                 mn_csr* elem_out, mn_csr* shared_out, mn_error_detail* err) {
  const NvtxScope range("mn_find_poly_neighbors");
  if (err) { err->elem = -1; err->pos = -1; }
  if (num_elems < 0 || conn_len < 0 || num_nodes < 0 || num_nodes > INT32_MAX) return MN_ERR_INVALID_ARG;
  if (num_elems > INT32_MAX || conn_len > INT32_MAX) return MN_ERR_CAPACITY;
  if (!d_off || (conn_len > 0 && !d_idx)) return MN_ERR_INVALID_ARG;
  if (!node_out && !elem_out && !shared_out) return MN_ERR_INVALID_ARG;
  Mem mem(a, (cudaStream_t)s);
  return poly_find(d_off, d_idx, num_elems, conn_len, num_nodes, mem, node_out, elem_out, shared_out, err);
}

mn_status mn_find_elem_neighbors(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N,
                                 const mn_allocator* a, mn_stream s, mn_csr* out, mn_error_detail* err) {
  return find(t, d_conn, M, N, a, s, false, true, nullptr, out, err);
}

mn_status mn_find_neighbors_both(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N,
                                 const mn_allocator* a, mn_stream s, mn_csr* no, mn_csr* eo,
                                 mn_error_detail* err) {
  return find(t, d_conn, M, N, a, s, true, true, no, eo, err);
}

mn_status mn_find_neighbors_both_chunked(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N,
                                         size_t max_workspace_bytes, const mn_allocator* a, mn_stream stream,
                                         mn_csr* no, mn_csr* eo, int64_t* chunks_used, mn_error_detail* err) {
  const NvtxScope range("mn_find_neighbors_both_chunked");
  if (err) { err->elem = -1; err->pos = -1; }
  mn_status st = check_args(t, d_conn, M, N);
  if (st != MN_OK) return st;
  if (!no || !eo) return MN_ERR_INVALID_ARG;
  Mem mem(a, (cudaStream_t)stream);
  const Plan P = make_plan(t, M, N);
  switch (t) {
    case MN_TRI3: return chunked_both<MN_TRI3>(P, d_conn, mem, max_workspace_bytes, chunks_used, no, eo, err);
    case MN_QUAD4: return chunked_both<MN_QUAD4>(P, d_conn, mem, max_workspace_bytes, chunks_used, no, eo, err);
    case MN_TET4: return chunked_both<MN_TET4>(P, d_conn, mem, max_workspace_bytes, chunks_used, no, eo, err);
    default: return chunked_both<MN_HEX8>(P, d_conn, mem, max_workspace_bytes, chunks_used, no, eo, err);
  }
}

mn_status mn_find_neighbors_both_host(mn_elem_type t, const int32_t* h_conn, int64_t M, int64_t N,
                                      const mn_allocator* dev_alloc, const mn_allocator* host_alloc,
                                      mn_stream stream, mn_csr* no, mn_csr* eo, mn_error_detail* err) {
  const NvtxScope range("mn_find_neighbors_both_host");
  mn_status st = check_args(t, h_conn, M, N);
  if (st != MN_OK) return st;
  if (!host_alloc || !host_alloc->alloc || !no || !eo) return MN_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  // side stream + event of the element-CSR D2H: per calling thread and per device
  static thread_local cudaStream_t sides[kMaxDevices] = {};
  static thread_local cudaEvent_t evs[kMaxDevices] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return MN_ERR_INVALID_ARG;
  cudaStream_t& side = sides[dev];
  cudaEvent_t& ev = evs[dev];
  if (!side && cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) return MN_ERR_CUDA;
  if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return MN_ERR_CUDA;
  Mem mem(dev_alloc, s);
  const int64_t Pe = (int64_t)M * arity_of(t);
  const size_t cbytes = (size_t)Pe * 4;
  std::memset(no, 0, sizeof(*no));
  std::memset(eo, 0, sizeof(*eo));
  // host outputs whose sizes are known up front
  no->owner = eo->owner = *host_alloc;
  no->num_nodes = eo->num_nodes = N;
  no->offsets = (int64_t*)host_alloc->alloc(host_alloc->ctx, (size_t)(N + 1) * 8, stream);
  eo->offsets = (int64_t*)host_alloc->alloc(host_alloc->ctx, (size_t)(N + 1) * 8, stream);
  eo->indices = Pe ? (int32_t*)host_alloc->alloc(host_alloc->ctx, (size_t)Pe * 4, stream) : nullptr;
  eo->nnz = Pe;
  mn_csr dn{}, de{};
  int32_t* d_conn = nullptr;
  HostSink sink{eo->offsets, eo->indices, side, ev, false};
  if (!no->offsets || !eo->offsets || (Pe && !eo->indices)) { st = MN_ERR_OOM; goto fail; }
  d_conn = (int32_t*)mem.get(cbytes);
  if (!d_conn) { st = MN_ERR_OOM; goto fail; }
  if (cbytes && cudaMemcpyAsync(d_conn, h_conn, cbytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
    st = MN_ERR_CUDA;
    goto fail;
  }
  st = find(t, d_conn, M, N, &mem.a, stream, true, true, &dn, &de, err, false, &sink);
  if (st != MN_OK) goto fail;
  if (!sink.issued &&   // (M == 0 returns before the sink point)
      cudaMemcpyAsync(eo->offsets, de.offsets, (size_t)(N + 1) * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
    st = MN_ERR_CUDA;
    goto fail;
  }
  no->nnz = dn.nnz;
  if (dn.nnz) {
    no->indices = (int32_t*)host_alloc->alloc(host_alloc->ctx, (size_t)dn.nnz * 4, stream);
    if (!no->indices) { st = MN_ERR_OOM; goto fail; }
  }
  if (cudaMemcpyAsync(no->offsets, dn.offsets, (size_t)(N + 1) * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      (dn.nnz && cudaMemcpyAsync(no->indices, dn.indices, (size_t)dn.nnz * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess))
    st = MN_ERR_CUDA;
  if (cudaStreamSynchronize(side) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) st = MN_ERR_CUDA;
  if (st != MN_OK) goto fail;
  mn_csr_release(&dn, stream);
  mn_csr_release(&de, stream);
  mem.put(d_conn);
  return MN_OK;
fail:
  cudaStreamSynchronize(side);
  cudaStreamSynchronize(s);
  mn_csr_release(&dn, stream);
  mn_csr_release(&de, stream);
  mem.put(d_conn);
  mn_csr_release(no, stream);
  mn_csr_release(eo, stream);
  return st;
}

// ---- pipelined host-buffer form (include/meshnbr.h mn_host_pipeline_*) ----
struct mn_host_pipeline {
  struct Ticket {
    int64_t id;
    int32_t* d_conn;
    mn_csr dn, de;
    cudaEvent_t done;
  };
  int device = 0;
  mn_allocator dev{}, host{};
  cudaStream_t up = nullptr, comp = nullptr, down = nullptr;
  cudaEvent_t ev_up = nullptr, ev_side = nullptr;
  std::vector<Ticket> inflight;
  int64_t next_id = 0;
  mn_status finish(Ticket& tk) {   // wait for the ticket's downloads, release its device buffers
    const bool ok = cudaEventSynchronize(tk.done) == cudaSuccess;
    cudaEventDestroy(tk.done);
    mn_csr_release(&tk.dn, (mn_stream)comp);
    mn_csr_release(&tk.de, (mn_stream)comp);
    if (tk.d_conn) dev.release(dev.ctx, tk.d_conn, (mn_stream)up);
    return ok ? MN_OK : MN_ERR_CUDA;
  }
};

mn_status mn_host_pipeline_create(const mn_allocator* dev_alloc, const mn_allocator* host_alloc,
                                  mn_host_pipeline** out) {
  if (!out || !host_alloc || !host_alloc->alloc) return MN_ERR_INVALID_ARG;
  *out = nullptr;
  auto* p = new (std::nothrow) mn_host_pipeline();
  if (!p) return MN_ERR_OOM;
  p->device = current_device();
  p->dev = dev_alloc && dev_alloc->alloc ? *dev_alloc : kDefaultAlloc;
  p->host = *host_alloc;
  if (cudaStreamCreateWithFlags(&p->up, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&p->down, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_up, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_side, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    mn_host_pipeline_destroy(p);
    return MN_ERR_CUDA;
  }
  *out = p;
  return MN_OK;
}

mn_status mn_host_pipeline_submit(mn_host_pipeline* p, mn_elem_type t, const int32_t* h_conn, int64_t M, int64_t N,
                                  mn_csr* no, mn_csr* eo, int64_t* ticket, mn_error_detail* err) {
  const NvtxScope range("mn_host_pipeline_submit");
  if (!p || !no || !eo || !ticket) return MN_ERR_INVALID_ARG;
  mn_status st = check_args(t, h_conn, M, N);
  if (st != MN_OK) return st;
  if (current_device() != p->device) return MN_ERR_INVALID_ARG;
  const int64_t Pe = (int64_t)M * arity_of(t);
  const size_t cbytes = (size_t)Pe * 4;
  std::memset(no, 0, sizeof(*no));
  std::memset(eo, 0, sizeof(*eo));
  mn_host_pipeline::Ticket tk{p->next_id, nullptr, {}, {}, nullptr};
  const mn_allocator& H = p->host;
  // host outputs whose sizes are known up front (the element CSR streams out during the node pass)
  no->owner = eo->owner = H;
  no->num_nodes = eo->num_nodes = N;
  no->offsets = (int64_t*)H.alloc(H.ctx, (size_t)(N + 1) * 8, (mn_stream)p->down);
  eo->offsets = (int64_t*)H.alloc(H.ctx, (size_t)(N + 1) * 8, (mn_stream)p->down);
  eo->indices = Pe ? (int32_t*)H.alloc(H.ctx, (size_t)Pe * 4, (mn_stream)p->down) : nullptr;
  eo->nnz = Pe;
  HostSink sink{eo->offsets, eo->indices, p->down, p->ev_side, false};
  if (!no->offsets || !eo->offsets || (Pe && !eo->indices)) { st = MN_ERR_OOM; goto fail; }
  if (cudaEventCreateWithFlags(&tk.done, cudaEventDisableTiming) != cudaSuccess) { st = MN_ERR_CUDA; goto fail; }
  // upload on its own stream: runs while the previous tickets' downloads are in flight
  tk.d_conn = (int32_t*)p->dev.alloc(p->dev.ctx, cbytes ? cbytes : 16, (mn_stream)p->up);
  if (!tk.d_conn) { st = MN_ERR_OOM; goto fail; }
  if ((cbytes && cudaMemcpyAsync(tk.d_conn, h_conn, cbytes, cudaMemcpyHostToDevice, p->up) != cudaSuccess) ||
      cudaEventRecord(p->ev_up, p->up) != cudaSuccess || cudaStreamWaitEvent(p->comp, p->ev_up, 0) != cudaSuccess) {
    st = MN_ERR_CUDA;
    goto fail;
  }
  st = find(t, tk.d_conn, M, N, &p->dev, (mn_stream)p->comp, true, true, &tk.dn, &tk.de, err, false, &sink);
  if (st != MN_OK) goto fail;
  // downloads: what the sink did not already send, after the compute stream's work
  if (cudaEventRecord(p->ev_side, p->comp) != cudaSuccess || cudaStreamWaitEvent(p->down, p->ev_side, 0) != cudaSuccess) {
    st = MN_ERR_CUDA;
    goto fail;
  }
  if (!sink.issued &&   // (M == 0 returns before the sink point)
      cudaMemcpyAsync(eo->offsets, tk.de.offsets, (size_t)(N + 1) * 8, cudaMemcpyDeviceToHost, p->down) != cudaSuccess) {
    st = MN_ERR_CUDA;
    goto fail;
  }
  no->nnz = tk.dn.nnz;
  if (tk.dn.nnz) {
    no->indices = (int32_t*)H.alloc(H.ctx, (size_t)tk.dn.nnz * 4, (mn_stream)p->down);
    if (!no->indices) { st = MN_ERR_OOM; goto fail; }
  }
  if (cudaMemcpyAsync(no->offsets, tk.dn.offsets, (size_t)(N + 1) * 8, cudaMemcpyDeviceToHost, p->down) != cudaSuccess ||
      (tk.dn.nnz &&
       cudaMemcpyAsync(no->indices, tk.dn.indices, (size_t)tk.dn.nnz * 4, cudaMemcpyDeviceToHost, p->down) != cudaSuccess) ||
      cudaEventRecord(tk.done, p->down) != cudaSuccess) {
    st = MN_ERR_CUDA;
    goto fail;
  }
  p->inflight.push_back(tk);
  *ticket = p->next_id++;
  return MN_OK;
fail:
  cudaStreamSynchronize(p->comp);
  cudaStreamSynchronize(p->down);
  cudaStreamSynchronize(p->up);
  mn_csr_release(&tk.dn, (mn_stream)p->comp);
  mn_csr_release(&tk.de, (mn_stream)p->comp);
  if (tk.d_conn) p->dev.release(p->dev.ctx, tk.d_conn, (mn_stream)p->up);
  if (tk.done) cudaEventDestroy(tk.done);
  mn_csr_release(no, (mn_stream)p->down);
  mn_csr_release(eo, (mn_stream)p->down);
  return st;
}

mn_status mn_host_pipeline_wait(mn_host_pipeline* p, int64_t ticket) {
  const NvtxScope range("mn_host_pipeline_wait");
  if (!p) return MN_ERR_INVALID_ARG;
  for (size_t i = 0; i < p->inflight.size(); ++i)
    if (p->inflight[i].id == ticket) {
      mn_host_pipeline::Ticket tk = p->inflight[i];
      p->inflight.erase(p->inflight.begin() + (std::ptrdiff_t)i);
      return p->finish(tk);
    }
  return MN_ERR_INVALID_ARG;
}

void mn_host_pipeline_destroy(mn_host_pipeline* p) {
  if (!p) return;
  for (auto& tk : p->inflight) p->finish(tk);
  p->inflight.clear();
  if (p->ev_up) cudaEventDestroy(p->ev_up);
  if (p->ev_side) cudaEventDestroy(p->ev_side);
  if (p->up) cudaStreamDestroy(p->up);
  if (p->comp) cudaStreamDestroy(p->comp);
  if (p->down) cudaStreamDestroy(p->down);
  delete p;
}

void mn_csr_release(mn_csr* c, mn_stream s) {
  if (!c) return;
  if (c->owner.release) {
    if (c->offsets) c->owner.release(c->owner.ctx, c->offsets, s);
    if (c->indices) c->owner.release(c->owner.ctx, c->indices, s);
  }
  std::memset(c, 0, sizeof(*c));
}

mn_status mn_workspace_bytes(mn_elem_type t, int64_t M, int64_t N, int modes, size_t* bytes) {
  mn_status st = check_args(t, (const void*)1, M, N);
  if (st != MN_OK || !bytes || modes < 1 || modes > 3) return MN_ERR_INVALID_ARG;
  const Plan P = make_plan(t, M, N);
  const bool wn = modes & 1, we = modes & 2;
  // mirrors pipeline_inc's arena (both element paths allocate the same pieces)
  Arena a;
  a.take<unsigned long long>(2);
  a.take<uint32_t>(32);
  a.take<unsigned int>(1);
  a.take<unsigned long long>((size_t)P.dp.nd * P.bins);
  a.take<uint64_t>((size_t)P.dp.nd * P.bins);
  a.take<uint64_t>((size_t)tiles_of(P.Pe, kTile) * P.bins);
  a.take<uint64_t>((size_t)tiles_of(P.N, kScanTile) + 1);
  a.take<int32_t>((size_t)P.N + 1);
  a.take<unsigned int>(1);
  a.take<int32_t>((size_t)P.N + 1);
  const size_t nch = (size_t)tiles_of(P.N, kChunkNodes);   // transpose: chunk counts, cursors, flag
  a.take<int32_t>(nch + 1);
  a.take<int32_t>(nch + 1);
  a.take<unsigned int>(1);
  if (g_elem_path.load() == 3) {   // MSD element path (forced only): range histogram, status, bases
    a.take<unsigned long long>(kMsdBins);
    a.take<uint64_t>((size_t)(tiles_of(P.Pe, kTile) ? tiles_of(P.Pe, kTile) : 1) * kMsdBins);
    a.take<uint64_t>(kMsdBins);
  }
  a.take<uint32_t>((size_t)P.N + 1);
  a.take<int64_t>(nch + 1);
  for (int i = 0; i < 4; ++i) a.take<uint32_t>((size_t)P.Pe);
  if (wn) {
    a.take<int32_t>((size_t)P.N);
    a.take<int32_t>((size_t)P.N);
    a.take<uint32_t>((size_t)P.N);
    if (!we) {
      a.take<int64_t>((size_t)P.N + 1);
      a.take<int32_t>((size_t)P.Pe);
    }
  }
  *bytes = a.off;
  return MN_OK;
}

size_t mn_chunk_workspace_bytes(mn_elem_type t, int64_t M, int64_t N, int64_t chunks) {
  if (t < 0 || t > 3 || M < 0 || N < 0 || chunks < 1) return 0;
  return chunk_workspace(make_plan(t, M, N), chunks);
}

mn_status mn_emit_node_pairs(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N, void* d_keys,
                             mn_stream stream, mn_error_detail* err) {
  if (err) { err->elem = -1; err->pos = -1; }
  mn_status st = check_args(t, d_conn, M, N);
  if (st != MN_OK) return st;
  if (M > 0 && !d_keys) return MN_ERR_INVALID_ARG;
  Mem mem(nullptr, (cudaStream_t)stream);
  switch (t) {
    case MN_TRI3: return emit_stage<MN_TRI3>(d_conn, M, N, d_keys, nullptr, nullptr, true, mem, err);
    case MN_QUAD4: return emit_stage<MN_QUAD4>(d_conn, M, N, d_keys, nullptr, nullptr, true, mem, err);
    case MN_TET4: return emit_stage<MN_TET4>(d_conn, M, N, d_keys, nullptr, nullptr, true, mem, err);
    default: return emit_stage<MN_HEX8>(d_conn, M, N, d_keys, nullptr, nullptr, true, mem, err);
  }
}

mn_status mn_emit_elem_pairs(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N, uint32_t* d_keys,
                             uint32_t* d_vals, mn_stream stream, mn_error_detail* err) {
  if (err) { err->elem = -1; err->pos = -1; }
  mn_status st = check_args(t, d_conn, M, N);
  if (st != MN_OK) return st;
  if (M > 0 && (!d_keys || !d_vals)) return MN_ERR_INVALID_ARG;
  Mem mem(nullptr, (cudaStream_t)stream);
  switch (t) {
    case MN_TRI3: return emit_stage<MN_TRI3>(d_conn, M, N, nullptr, d_keys, d_vals, false, mem, err);
    case MN_QUAD4: return emit_stage<MN_QUAD4>(d_conn, M, N, nullptr, d_keys, d_vals, false, mem, err);
    case MN_TET4: return emit_stage<MN_TET4>(d_conn, M, N, nullptr, d_keys, d_vals, false, mem, err);
    default: return emit_stage<MN_HEX8>(d_conn, M, N, nullptr, d_keys, d_vals, false, mem, err);
  }
}

mn_status mn_radix_sort_keys(void* d_keys, int key_bytes, int64_t n, int key_bits, const mn_allocator* a,
                             mn_stream stream) {
  if (n < 0 || (n > 0 && !d_keys) || (key_bytes != 4 && key_bytes != 8) || key_bits < 0 ||
      key_bits > 8 * key_bytes)
    return MN_ERR_INVALID_ARG;
  Mem mem(a, (cudaStream_t)stream);
  if (key_bytes == 8) return lsd_sort<uint64_t, false>((uint64_t*)d_keys, nullptr, n, key_bits, mem);
  return lsd_sort<uint32_t, false>((uint32_t*)d_keys, nullptr, n, key_bits, mem);
}

mn_status mn_radix_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_vals, int64_t n, int key_bits,
                                  const mn_allocator* a, mn_stream stream) {
  if (n < 0 || (n > 0 && (!d_keys || !d_vals)) || key_bits < 0 || key_bits > 32) return MN_ERR_INVALID_ARG;
  Mem mem(a, (cudaStream_t)stream);
  return lsd_sort<uint32_t, true>(d_keys, d_vals, n, key_bits, mem);
}

mn_status mn_unique_node_csr(const void* d_sorted_keys, int key_bytes, int64_t n, int64_t N,
                             int64_t* d_offsets, int32_t* d_indices, int64_t* h_nnz,
                             const mn_allocator* a, mn_stream stream) {
  if (n < 0 || N < 0 || N > INT32_MAX || !d_offsets || !h_nnz || (n > 0 && (!d_sorted_keys || !d_indices)) ||
      (key_bytes != 4 && key_bytes != 8))
    return MN_ERR_INVALID_ARG;
  Mem mem(a, (cudaStream_t)stream);
  const int b = node_bits(N);
  if (key_bytes == 8) return unique_csr<uint64_t>((const uint64_t*)d_sorted_keys, n, b, N, d_offsets, d_indices, h_nnz, mem);
  return unique_csr<uint32_t>((const uint32_t*)d_sorted_keys, n, b, N, d_offsets, d_indices, h_nnz, mem);
}

mn_status mn_elem_offsets(const uint32_t* d_sorted_keys, int64_t n, int64_t N, int64_t* d_offsets,
                          mn_stream stream) {
  if (n < 0 || N < 0 || !d_offsets || (n > 0 && !d_sorted_keys)) return MN_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return cudaMemsetAsync(d_offsets, 0, (size_t)(N + 1) * 8, s) == cudaSuccess ? MN_OK : MN_ERR_CUDA;
  cudaError_t e = launch("elem_offsets", 4.0 * n + 8.0 * (N + 1), s, [&] {
    k_elem_offsets<false><<<stream_grid(n / 4 + 1), 256, 0, s>>>(d_sorted_keys, n, N, d_offsets, nullptr);
  });
  return e == cudaSuccess ? MN_OK : MN_ERR_CUDA;
}

mn_status mn_exclusive_scan_i32(const int32_t* d_counts, int64_t n, int64_t* d_out, const mn_allocator* a,
                                mn_stream stream) {
  if (n < 0 || !d_out || (n > 0 && !d_counts)) return MN_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return cudaMemsetAsync(d_out, 0, 8, s) == cudaSuccess ? MN_OK : MN_ERR_CUDA;
  Mem mem(a, s);
  const int64_t tiles = tiles_of(n, kScanTile);
  const size_t bytes = 256 + (size_t)tiles * 8;
  char* ws = (char*)mem.get(bytes);
  if (!ws) return MN_ERR_OOM;
  mn_status st = MN_OK;
  uint32_t* ticket = (uint32_t*)ws;
  uint64_t* status = (uint64_t*)(ws + 256);
  if (cudaMemsetAsync(ws, 0, bytes, s) != cudaSuccess) st = MN_ERR_CUDA;
  if (st == MN_OK &&
      launch("scan_i32", 4.0 * n + 8.0 * (n + 1), s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles, kScanThreads, 0, s>>>(d_counts, n, d_out, status, ticket, 1);
      }) != cudaSuccess)
    st = MN_ERR_CUDA;
  mem.put(ws);
  return st;
}

mn_status mn_dist_bucket(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t base, int64_t N, int world,
                         int self_rank, uint64_t* d_pairs, int64_t* h_counts, int32_t** d_row_elems,
                         int32_t** d_rows, int64_t* h_row_counts, const mn_allocator* a, mn_stream stream,
                         mn_error_detail* err) {
  if (err) { err->elem = -1; err->pos = -1; }
  mn_status st = check_args(t, d_conn, M, N);
  if (st != MN_OK) return st;
  if (world < 1 || world > 512 || self_rank < 0 || self_rank >= world || !h_counts || !h_row_counts ||
      !d_row_elems || !d_rows || base < 0 || (M > 0 && !d_pairs))
    return MN_ERR_INVALID_ARG;
  if (base + M > INT32_MAX) return MN_ERR_CAPACITY;
  *d_row_elems = nullptr;
  *d_rows = nullptr;
  Mem mem(a, (cudaStream_t)stream);
#define MN_DB(TT)                                                                                      \
  return world <= 256                                                                                  \
             ? dist_bucket_impl<TT, 256>(d_conn, M, base, N, world, self_rank, d_pairs, h_counts,    \
                                         d_row_elems, d_rows, h_row_counts, mem, err)                \
             : dist_bucket_impl<TT, 512>(d_conn, M, base, N, world, self_rank, d_pairs, h_counts,    \
                                         d_row_elems, d_rows, h_row_counts, mem, err)
  switch (t) {
    case MN_TRI3: MN_DB(MN_TRI3);
    case MN_QUAD4: MN_DB(MN_QUAD4);
    case MN_TET4: MN_DB(MN_TET4);
    default: MN_DB(MN_HEX8);
  }
#undef MN_DB
}

mn_status mn_dist_finish(mn_elem_type t, const uint64_t* d_pairs, int64_t n, const int32_t* d_row_elems,
                         const int32_t* d_rows, int64_t n_rows, const int32_t* d_conn_shard, int64_t shard_elems,
                         int64_t global_elem_base, int64_t N, int64_t lo, int64_t hi, const mn_allocator* a,
                         mn_stream stream, mn_csr* node_slice, mn_csr* elem_slice) {
  if (t < 0 || t > 3 || n < 0 || n_rows < 0 || shard_elems < 0 || N < 0 || N > INT32_MAX || lo < 0 || hi < lo ||
      hi > N || !node_slice || !elem_slice || (n > 0 && !d_pairs) || (n_rows > 0 && (!d_row_elems || !d_rows)) ||
      (shard_elems > 0 && !d_conn_shard) || n > INT32_MAX)
    return MN_ERR_INVALID_ARG;
  Mem mem(a, (cudaStream_t)stream);
#define MN_DF(TT)                                                                                          \
  return dist_finish_impl<TT>(pair_src(d_pairs, n), n, d_row_elems, d_rows, n_rows, d_conn_shard, global_elem_base,   \
                              shard_elems, N, lo, hi, mem, node_slice, elem_slice)
  switch (t) {
    case MN_TRI3: MN_DF(MN_TRI3);
    case MN_QUAD4: MN_DF(MN_QUAD4);
    case MN_TET4: MN_DF(MN_TET4);
    default: MN_DF(MN_HEX8);
  }
#undef MN_DF
}

mn_status mn_find_neighbors_dist(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t base, int64_t N,
                                 const mn_comm* comm, const mn_allocator* a, mn_stream stream, mn_csr* node_slice,
                                 mn_csr* elem_slice, mn_dist_info* info, mn_error_detail* err) {
  const NvtxScope range("mn_find_neighbors_dist");
  if (err) { err->elem = -1; err->pos = -1; }
  if (t < 0 || t > 3 || M < 0 || N < 0 || N > INT32_MAX || base < 0 || !comm || !comm->allgather ||
      !comm->alltoallv || comm->world < 1 || comm->world > 512 || comm->rank < 0 || comm->rank >= comm->world ||
      !node_slice || !elem_slice || (M > 0 && !d_conn))
    return MN_ERR_INVALID_ARG;
  if (base + M > INT32_MAX) return MN_ERR_CAPACITY;
  if (info) std::memset(info, 0, sizeof(*info));
  Mem mem(a, (cudaStream_t)stream);
  return dist2_dispatch(t, d_conn, M, base, N, comm, nullptr, mem, node_slice, elem_slice, info, err);
}

mn_status mn_symm_create(const mn_comm* comm, size_t initial_bytes, mn_symm** out) {
  if (!comm || !out || !comm->allgather || comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world)
    return MN_ERR_INVALID_ARG;
  mn_symm* h = new (std::nothrow) mn_symm();
  if (!h) return MN_ERR_OOM;
  h->comm = *comm;
  h->dev = current_device();
  h->peer.assign(comm->world, nullptr);
  const mn_status st = initial_bytes ? symm_reserve(h, initial_bytes, nullptr) : MN_OK;
  if (st != MN_OK) { mn_symm_destroy(h); return st; }
  *out = h;
  return MN_OK;
}

mn_status mn_symm_unmap(mn_symm* h) {
  if (!h) return MN_ERR_INVALID_ARG;
  for (int g = 0; g < (int)h->peer.size(); ++g) {
    if (g != h->comm.rank && h->peer[g]) cudaIpcCloseMemHandle(h->peer[g]);
    if (g != h->comm.rank) h->peer[g] = nullptr;
  }
  h->cap = 0;   // a later call re-maps (collectively) before any use
  return MN_OK;
}

mn_status mn_symm_destroy(mn_symm* h) {
  if (!h) return MN_ERR_INVALID_ARG;
  mn_symm_unmap(h);
  if (h->local) cudaFree(h->local);
  delete h;
  return MN_OK;
}

size_t mn_symm_capacity(const mn_symm* h) { return h ? h->cap : 0; }

mn_status mn_find_neighbors_dist_p2p(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t base, int64_t N,
                                     mn_symm* symm, const mn_allocator* a, mn_stream stream, mn_csr* node_slice,
                                     mn_csr* elem_slice, mn_dist_info* info, mn_error_detail* err) {
  const NvtxScope range("mn_find_neighbors_dist_p2p");
  if (err) { err->elem = -1; err->pos = -1; }
  if (t < 0 || t > 3 || M < 0 || N < 0 || N > INT32_MAX || base < 0 || !symm || !node_slice || !elem_slice ||
      (M > 0 && !d_conn) || symm->comm.world > 512)
    return MN_ERR_INVALID_ARG;
  if (base + M > INT32_MAX) return MN_ERR_CAPACITY;
  if (info) std::memset(info, 0, sizeof(*info));
  Mem mem(a, (cudaStream_t)stream);
  return dist2_dispatch(t, d_conn, M, base, N, &symm->comm, symm, mem, node_slice, elem_slice, info, err);
}

static mn_status dist_one(bool node, mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t base, int64_t N,
                          void* nccl_comm, const mn_allocator* a, mn_stream stream, mn_csr* slice, int64_t* lo,
                          int64_t* hi, int64_t* gbase, mn_error_detail* err) {
  if (!slice) return MN_ERR_INVALID_ARG;
  mn_comm c{};
  mn_status st = mn_comm_from_nccl(nccl_comm, &c);
  if (st != MN_OK) return st;
  mn_csr ns{}, es{};
  mn_dist_info info{};
  st = mn_find_neighbors_dist(t, d_conn, M, base, N, &c, a, stream, &ns, &es, &info, err);
  if (st != MN_OK) return st;
  if (node) { *slice = ns; mn_csr_release(&es, stream); } else { *slice = es; mn_csr_release(&ns, stream); }
  if (lo) *lo = info.lo;
  if (hi) *hi = info.hi;
  if (gbase) *gbase = node ? info.node_base : info.elem_base;
  return MN_OK;
}

mn_status mn_find_node_neighbors_dist(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t base, int64_t N,
                                      void* nccl_comm, const mn_allocator* a, mn_stream stream, mn_csr* slice,
                                      int64_t* lo, int64_t* hi, int64_t* gbase, mn_error_detail* err) {
  return dist_one(true, t, d_conn, M, base, N, nccl_comm, a, stream, slice, lo, hi, gbase, err);
}

mn_status mn_find_elem_neighbors_dist(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t base, int64_t N,
                                      void* nccl_comm, const mn_allocator* a, mn_stream stream, mn_csr* slice,
                                      int64_t* lo, int64_t* hi, int64_t* gbase, mn_error_detail* err) {
  return dist_one(false, t, d_conn, M, base, N, nccl_comm, a, stream, slice, lo, hi, gbase, err);
}

int mn_nccl_available(void) { return nccl().ok ? 1 : 0; }

mn_status mn_nccl_get_unique_id(void* id128) {
  if (!id128) return MN_ERR_INVALID_ARG;
  const NcclApi& n = nccl();
  if (!n.ok) return MN_ERR_COMM;
  ncclUniqueId id;
  if (n.get_unique_id(&id) != ncclSuccess) return MN_ERR_COMM;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof(id));
  return MN_OK;
}

mn_status mn_nccl_comm_init(const void* id128, int world, int rank, void** nccl_comm) {
  if (!id128 || !nccl_comm || world < 1 || rank < 0 || rank >= world) return MN_ERR_INVALID_ARG;
  const NcclApi& n = nccl();
  if (!n.ok) return MN_ERR_COMM;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  if (n.comm_init_rank(&c, world, id, rank) != ncclSuccess) return MN_ERR_COMM;
  *nccl_comm = c;
  return MN_OK;
}

mn_status mn_nccl_comm_destroy(void* nccl_comm) {
  if (!nccl_comm) return MN_ERR_INVALID_ARG;
  const NcclApi& n = nccl();
  if (!n.ok) return MN_ERR_COMM;
  return n.comm_destroy((ncclComm_t)nccl_comm) == ncclSuccess ? MN_OK : MN_ERR_COMM;
}

mn_status mn_comm_from_nccl(void* nccl_comm, mn_comm* out) {
  if (!nccl_comm || !out) return MN_ERR_INVALID_ARG;
  const NcclApi& n = nccl();
  if (!n.ok) return MN_ERR_COMM;
  int world = 0, rank = 0;
  if (n.comm_count((ncclComm_t)nccl_comm, &world) != ncclSuccess ||
      n.comm_user_rank((ncclComm_t)nccl_comm, &rank) != ncclSuccess)
    return MN_ERR_COMM;
  out->rank = rank;
  out->world = world;
  out->ctx = nccl_comm;
  out->allgather = nccl_allgather_cb;
  out->alltoallv = nccl_alltoallv_cb;
  return MN_OK;
}

mn_status mn_dist_plan(int world, int rank, const int64_t* gathered, int64_t* recv_counts, int64_t* recv_row_counts,
                       mn_error_detail* err) {
  if (err) { err->elem = -1; err->pos = -1; }
  if (world < 1 || rank < 0 || rank >= world || !gathered || !recv_counts || !recv_row_counts)
    return MN_ERR_INVALID_ARG;
  return dist_plan(world, rank, gathered, recv_counts, recv_row_counts, err);
}

mn_status mn_memcpy_sync(void* dst, const void* src, size_t bytes, mn_stream stream) {
  if (bytes == 0) return MN_OK;
  if (!dst || !src) return MN_ERR_INVALID_ARG;
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream) != cudaSuccess ||
      cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) {
    cudaGetLastError();
    return MN_ERR_CUDA;
  }
  return MN_OK;
}

int64_t mn_launch_count(void) { return g_launches.load(); }

mn_status mn_set_elem_path(int mode) {
  if (mode < 0 || mode > 3) return MN_ERR_INVALID_ARG;
  g_elem_path.store(mode);
  return MN_OK;
}

int mn_get_elem_path(void) { return g_elem_path.load(); }

mn_status mn_time_both(mn_elem_type t, const int32_t* d_conn, int64_t M, int64_t N, int reps, mn_stream stream,
                       double* median_us, double* min_us) {
  const NvtxScope range("mn_time_both");
  if (reps < 1 || !median_us) return MN_ERR_INVALID_ARG;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, current_device()) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;   // keep freed blocks in the pool between calls
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  std::vector<double> us;
  for (int r = 0; r < reps + 2; ++r) {   // 2 warm-up calls
    mn_csr no{}, eo{};
    const auto t0 = std::chrono::steady_clock::now();
    const mn_status st = mn_find_neighbors_both(t, d_conn, M, N, nullptr, stream, &no, &eo, nullptr);
    if (st != MN_OK) return st;
    // the call returns with its last kernel (the node compaction) still queued: wait for it
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return MN_ERR_CUDA;
    const auto t1 = std::chrono::steady_clock::now();
    mn_csr_release(&no, stream);
    mn_csr_release(&eo, stream);
    if (r >= 2) us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(us.begin(), us.end());
  *median_us = us[us.size() / 2];
  if (min_us) *min_us = us.front();
  return MN_OK;
}

mn_status mn_set_small_path(int64_t max_incidences) {
  if (max_incidences < 0) return MN_ERR_INVALID_ARG;
  g_small_max.store(std::min<int64_t>(max_incidences, kSmallMaxPe));
  return MN_OK;
}


mn_status mn_set_chunk_cap(int cap) {
  if (cap < 0) return MN_ERR_INVALID_ARG;
  g_chunk_cap.store(cap);
  return MN_OK;
}

void mn_profile_enable(int on) { g_prof = on != 0; }

void mn_profile_reset(void) {
  for (auto& r : g_recs) { g_evpool.push_back(r.a); g_evpool.push_back(r.b); }
  g_recs.clear();
  g_table.clear();
}

int mn_profile_collect(void) {
  g_table.clear();
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    ProfEntry* e = nullptr;
    for (auto& x : g_table)
      if (x.name == r.name) { e = &x; break; }
    if (!e) { g_table.push_back({r.name, 0, 0.0, 0.0}); e = &g_table.back(); }
    e->launches += 1;
    e->ms += ms;
    e->bytes += r.bytes;
  }
  return (int)g_table.size();
}

mn_status mn_profile_entry(int i, const char** name, int64_t* launches, double* total_ms, double* alg_bytes) {
  if (i < 0 || i >= (int)g_table.size()) return MN_ERR_INVALID_ARG;
  if (name) *name = g_table[i].name.c_str();
  if (launches) *launches = g_table[i].launches;
  if (total_ms) *total_ms = g_table[i].ms;
  if (alg_bytes) *alg_bytes = g_table[i].bytes;
  return MN_OK;
}

}  // extern "C"
