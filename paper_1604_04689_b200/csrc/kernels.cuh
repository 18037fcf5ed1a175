// kernels.cuh — the hot-path kernels of libmeshnbr (sm_100a).
//
// Method (§2.2.1, §2.2.2): create (node, neighbour) and (node,
// element) integer pairs, sort them by the first integer, then segmented reduction + scan give
// each vertex's count and first index.  B200 design (DESIGN.md §"Kernels"):
//   k_hist_validate   validate conn + digit histograms of the node ids (one read of conn)
//   k_bucket_bases    per-pass global digit bucket bases (exclusive scan of the histograms)
//   k_onesweep        one LSD digit pass: warp-match ranking, decoupled look-back, smem scatter;
//                     pass 0 creates the pairs from conn on the fly (no emitted-pair round trip)
//   k_unique_node     fused adjacent-difference dedupe + compaction + run length -> offsets
//   k_elem_offsets    run starts of the sorted element-pair keys -> offsets
//   k_scan_i32        single-pass look-back exclusive scan (standalone row a5)
#pragma once
#include <type_traits>

#include "common.cuh"

namespace mn {

// ================================================================================================
// Digit plan.  A node id of b bits is split into nd digits (widths w_j, shifts s_j).  Node keys
// (a << b | v) are sorted LSD over the v digits then the a digits; element keys (node) over the nd
// digits.  Because every local node of a TRI3/QUAD4/TET4/HEX8 element has the same number C of
// incident element edges, the histogram of any node-key digit equals C x the histogram of that
// digit over the conn entries — so one pass over conn yields every pass's bucket sizes.
// ================================================================================================
struct DigitPlan {
  int nd;
  int shift[4];
  int width[4];
};

struct PassDigit {   // digit(key) = OWNER ? (key >> shift) / div : (key >> shift) & mask
  int shift;
  uint32_t mask;
  uint64_t div;
};

template <typename KeyT, bool OWNER>
__device__ __forceinline__ uint32_t digit_of(KeyT key, const PassDigit& pd, uint32_t maxbin) {
  if (OWNER && sizeof(KeyT) == 4) {   // 32-bit keys (node ids; div <= N < 2^31): 32-bit division
    const uint32_t d = ((uint32_t)key >> pd.shift) / (uint32_t)pd.div;
    return d > maxbin ? maxbin : d;
  } else if (OWNER) {
    uint64_t d = ((uint64_t)key >> pd.shift) / pd.div;
    return d > maxbin ? maxbin : (uint32_t)d;
  } else {
    return (uint32_t)(key >> pd.shift) & pd.mask;
  }
}

// ================================================================================================
// k_hist_validate: one thread per element.  Validation (reading R8) + per-digit histograms of the
// node ids of valid elements.  Histograms are CTA-private in shared memory, flushed once.
// ================================================================================================
template <int T, bool ALIGNED, bool RAND = false>
__device__ __forceinline__ void load_row(const int32_t* __restrict__ conn, int64_t e, int (&row)[Elem<T>::K]);

// The warp walks 32 consecutive elements per step.  A digit that is the same in all 32 lanes
// (typical for the high digits of a mesh numbered with spatial locality) is counted with one
// shared-memory atomic instead of 32 (__reduce_min/max_sync test).
template <int T, int BINS, bool ALIGNED>
__global__ void __launch_bounds__(256)
k_hist_validate(const int32_t* __restrict__ conn, int64_t M, int64_t N, int64_t elem_base,
                DigitPlan dp, int owner_hist, uint64_t owner_div,
                unsigned long long* __restrict__ hist, unsigned long long* __restrict__ err) {
  constexpr int K = Elem<T>::K;
  __shared__ uint32_t sh[4 * BINS];
  const int nh = owner_hist ? 1 : dp.nd;
  for (int i = threadIdx.x; i < nh * BINS; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < M; base += stride) {
    const int64_t e = base + lane;
    const bool in = e < M;
    int v[K];
    if (in) {
      load_row<T, ALIGNED>(conn, e, v);
    } else {
#pragma unroll
      for (int p = 0; p < K; ++p) v[p] = 0;
    }
    int kind = 0;
    const int bad = in ? row_bad<K>(v, (uint32_t)N, kind) : -1;
    if (in) {
      if (bad >= 0) atomicMin(err, (unsigned long long)err_encode((uint64_t)(elem_base + e), kind, bad));
    }
    const bool ok = in && bad < 0;
    const unsigned okm = __ballot_sync(FULL, ok);
    if (owner_hist) {
      if (ok) {
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const uint64_t d = owner_div <= 0xFFFFFFFFull ? (uint64_t)((uint32_t)v[p] / (uint32_t)owner_div)
                                                        : (uint64_t)v[p] / owner_div;
          atomicAdd(&sh[d < BINS ? d : BINS - 1], 1u);
        }
      }
      continue;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= dp.nd) break;
      const int sh_j = dp.shift[j];
      const uint32_t mk = (1u << dp.width[j]) - 1u;
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const uint32_t dg = ((uint32_t)v[p] >> sh_j) & mk;
        if (j > 0 && okm == FULL) {   // the lowest digit is practically never warp-uniform
          const uint32_t d0 = __shfl_sync(FULL, dg, 0);
          if (__all_sync(FULL, dg == d0)) {
            if (lane == 0) atomicAdd(&sh[j * BINS + d0], 32u);
            continue;
          }
        }
        if (ok) atomicAdd(&sh[j * BINS + dg], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nh * BINS; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// Histograms of arbitrary keys (generic sort entry point): all digits of 8 bits.
template <typename KeyT>
__global__ void __launch_bounds__(256)
k_hist_keys(const KeyT* __restrict__ keys, int64_t n, int ndig, unsigned long long* __restrict__ hist) {
  __shared__ uint32_t sh[8 * 256];
  for (int i = threadIdx.x; i < ndig * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    KeyT k = keys[i];
    for (int j = 0; j < ndig; ++j) atomicAdd(&sh[j * 256 + (uint32_t)((k >> (8 * j)) & 0xFF)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ndig * 256; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// ================================================================================================
// k_bucket_bases: block q computes bases[q][d] = mult_q * sum_{d' < d} hist[hidx_q][d'].
// ================================================================================================
struct BasesDesc {
  int npass;
  int hidx[16];
  int mult[16];
};

template <int BINS>
__global__ void __launch_bounds__(BINS)
k_bucket_bases(const unsigned long long* __restrict__ hist, BasesDesc bd, uint64_t* __restrict__ bases,
               const unsigned long long* __restrict__ err) {
  if (err && *err != ERR_NONE) return;
  __shared__ uint64_t wsum[BINS / 32];
  const int q = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint64_t x = (uint64_t)bd.mult[q] * hist[bd.hidx[q] * BINS + t];
  uint64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  uint64_t pre = 0;
  for (int i = 0; i < w; ++i) pre += wsum[i];
  bases[q * BINS + t] = pre + inc - x;
}

// ================================================================================================
// k_onesweep: one stable LSD digit pass (onesweep).
//   SRC 0: keys (and values) from arrays
//   SRC 1: node pair keys (a << b | v) created from conn on the fly (slot order e*2E + r)
//   SRC 2: element pair keys conn[i] with value i / K created from conn on the fly
//   SRC 3: element pairs packed (node << 32 | elem_base + i / K) created from conn (dist bucketing)
// Tile = THREADS*ITEMS items in warp-striped order (warp w owns a contiguous 32*ITEMS chunk, item
// i of lane l is chunk[i*32 + l]), so the per-warp running histogram ranks keys stably.
// ================================================================================================
struct PassArgs {
  const void* keys_in;
  void* keys_out;
  const uint32_t* vals_in;
  uint32_t* vals_out;
  const int32_t* conn;
  int node_bits;       // SRC 1: b
  int64_t elem_base;   // SRC 3
  int64_t n;
  PassDigit pd;
  const uint64_t* bases;   // [BINS]
  uint64_t* status;        // [tiles][BINS]
  uint32_t* ticket;
  uint32_t epoch;
  const unsigned long long* err;
  int32_t* counts;         // COUNTS mode: per-key run lengths (last element pass)
  // P2P (fused multi-GPU bucketing, SRC 3): the items of owner digit d are stored at dst[d] + their
  // rank in the bucket — a region of rank d's receive buffer, reached over NVLink peer memory — and
  // for d != self the element's row goes to rowdst[d] + rank * K (rank d's row table)
  uint64_t* const* dst;
  int32_t* const* rowdst;
  int self;
};

template <int THREADS, int ITEMS, int BINS>
struct OnesweepSmem {
  static constexpr int WARPS = THREADS / 32;
  uint32_t whist[WARPS][BINS];
  uint32_t ecnt[BINS];   // EARLY: tile digit counts from shared-memory atomics, before ranking
  uint32_t binstart[BINS];
  uint64_t gofs[BINS];
  uint64_t wsum[WARPS];
  uint32_t tile;
};

// Peer mask of lanes holding the same digit.  RANK 0: __match_any_sync.  RANK 1: one ballot per
// digit bit (vote unit only, no scoreboard wait).  RANK 2: RANK 1 behind a warp-uniform test.
template <int RANK, int BINS>
__device__ __forceinline__ unsigned digit_peers(uint32_t d) {
  constexpr int RB = BINS >= 512 ? 9 : 8;
  if (RANK == 0) return __match_any_sync(FULL, d);
  if (RANK == 2) {
    const uint32_t d0 = __shfl_sync(FULL, d, 0);
    if (__all_sync(FULL, d == d0)) return FULL;
  }
  unsigned peers = FULL;
#pragma unroll
  for (int bit = 0; bit < RB; ++bit) {
    const bool set = (d >> bit) & 1u;
    const unsigned bal = __ballot_sync(FULL, set);
    peers &= set ? bal : ~bal;
  }
  return peers;
}

// COUNTS (last pass of the element sort): the sorted keys are not written; instead each run of
// equal keys inside the tile adds its length to counts[key] with two atomics (+end+1 at the run's
// last slot, -start at its first), so counts[] ends as the per-node incidence counts whose
// exclusive scan is the element-CSR offsets.
// EARLY: the tile histogram is built first with shared-memory atomics, the aggregate published and
// the first look-back window requested before the (slower) stable ranking, so the look-back round
// trip overlaps the ranking instead of following it (the "early counts" of onesweep).
template <typename KeyT, int SRC, int T, bool PAYLOAD, bool OWNER, int BINS, int THREADS, int ITEMS,
          int W = 4, int MINB = 3, int RANK = 0, bool COUNTS = false, bool EARLY = false, bool P2P = false>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep(PassArgs pa) {
  constexpr int WARPS = THREADS / 32;
  constexpr int TILE = THREADS * ITEMS;
  // digits owned per thread (contiguous); with BINS < THREADS only threads tid < BINS own one
  constexpr int BPT = BINS >= THREADS ? BINS / THREADS : 1;
  static_assert(BINS % THREADS == 0 || THREADS % BINS == 0, "BINS and THREADS must nest");
  using Sm = OnesweepSmem<THREADS, ITEMS, BINS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
  KeyT* skeys = reinterpret_cast<KeyT*>(smem_raw + ((sizeof(Sm) + 15) & ~size_t(15)));
  uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + TILE);

  if (*pa.err != ERR_NONE) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool own = BINS >= THREADS || tid < BINS;   // warp-uniform
  if (tid == 0) sm.tile = atomicAdd(pa.ticket, 1u);
  for (int i = tid; i < WARPS * BINS; i += THREADS) (&sm.whist[0][0])[i] = 0;
  if (EARLY)
    for (int i = tid; i < BINS; i += THREADS) sm.ecnt[i] = 0;
  __syncthreads();
  const uint32_t tile = sm.tile;
  const int64_t base = (int64_t)tile * TILE;
  const int64_t chunk = base + (int64_t)warp * 32 * ITEMS;

  // ---- load (pair creation for pass 0) ----
  KeyT key[ITEMS];
  uint32_t val[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = chunk + i * 32 + lane;
    val[i] = 0;
    if (idx < pa.n) {
      if (SRC == 0) {
        key[i] = ld_stream(reinterpret_cast<const KeyT*>(pa.keys_in) + idx);
        if (PAYLOAD) val[i] = ld_stream(pa.vals_in + idx);
      } else if (SRC == 1) {
        constexpr int K = Elem<T>::K, S = 2 * Elem<T>::E;
        const int64_t e = idx / S;
        const int r = (int)(idx - e * S);
        int la, lb;
        slot_locals<T>(r, la, lb);
        const uint32_t a = (uint32_t)__ldg(pa.conn + e * K + la);
        const uint32_t v = (uint32_t)__ldg(pa.conn + e * K + lb);
        key[i] = (KeyT)(((KeyT)a << pa.node_bits) | (KeyT)v);
      } else if (SRC == 2) {
        constexpr int K = Elem<T>::K;
        key[i] = (KeyT)(uint32_t)__ldg(pa.conn + idx);
        val[i] = (uint32_t)(idx / K);
      } else {
        constexpr int K = Elem<T>::K;
        key[i] = (KeyT)(((uint64_t)(uint32_t)__ldg(pa.conn + idx) << 32) |
                        (uint64_t)(pa.elem_base + idx / K));
      }
    } else {
      key[i] = (KeyT)~(KeyT)0;
    }
  }

  // ---- EARLY: tile histogram, aggregate published, first look-back window in flight ----
  uint64_t lbw[BPT][W];
  if (EARLY) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t idx = chunk + i * 32 + lane;
      if (idx < pa.n) atomicAdd(&sm.ecnt[digit_of<KeyT, OWNER>(key[i], pa.pd, BINS - 1)], 1u);
    }
    __syncthreads();
    if (own) {
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        const int b = tid * BPT + j;
        st_relaxed_u64(pa.status + (size_t)tile * BINS + b,
                       st_pack(pa.epoch, tile == 0 ? ST_INC : ST_AGG, sm.ecnt[b]));
      }
      if (tile > 0) lookback_issue<BPT, W>(pa.status, BINS, tile, tid * BPT, lbw);
    }
  }

  // ---- rank: per-warp running digit histogram, warp-match aggregated; dr = digit | rank << 16 ----
  uint32_t dr[ITEMS];
  if (RANK == 3) {
    // all MATCHes first (independent, pipelined), then the per-warp histogram chain
    unsigned pm[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t idx = chunk + i * 32 + lane;
      dr[i] = idx < pa.n ? digit_of<KeyT, OWNER>(key[i], pa.pd, BINS - 1) : (uint32_t)(BINS - 1);
      pm[i] = __match_any_sync(FULL, dr[i]);
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t d = dr[i];
      const int leader = __ffs(pm[i]) - 1;
      uint32_t old = 0;
      if (lane == leader) {
        old = sm.whist[warp][d];
        sm.whist[warp][d] = old + __popc(pm[i]);
      }
      old = __shfl_sync(FULL, old, leader);
      dr[i] = d | ((old + __popc(pm[i] & lanemask_lt())) << 16);
      __syncwarp();   // orders this leader's histogram write before the next item's read by another lane
    }
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t idx = chunk + i * 32 + lane;
      const uint32_t d = idx < pa.n ? digit_of<KeyT, OWNER>(key[i], pa.pd, BINS - 1) : (uint32_t)(BINS - 1);
      const unsigned peers = digit_peers<RANK, BINS>(d);
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (lane == leader) {
        old = sm.whist[warp][d];
        sm.whist[warp][d] = old + __popc(peers);
      }
      old = __shfl_sync(FULL, old, leader);
      dr[i] = d | ((old + __popc(peers & lanemask_lt())) << 16);
      __syncwarp();   // (as above)
    }
  }
  __syncthreads();

  // ---- tile digit counts; publish the aggregate (tile 0: the inclusive prefix) ----
  const int64_t nvalid64 = pa.n - base;
  const int nvalid = nvalid64 >= TILE ? TILE : (int)nvalid64;
  uint32_t cnt[BPT];
  uint32_t tsum = 0;
#pragma unroll
  for (int j = 0; j < BPT; ++j) {
    cnt[j] = 0;
    if (!own) continue;
    const int b = tid * BPT + j;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t t = sm.whist[w][b];
      sm.whist[w][b] = run;
      run += t;
    }
    cnt[j] = run;
    tsum += run;
    if (!EARLY) {
      const uint32_t pub = (b == BINS - 1) ? run - (uint32_t)(TILE - nvalid) : run;
      st_relaxed_u64(pa.status + (size_t)tile * BINS + b, st_pack(pa.epoch, tile == 0 ? ST_INC : ST_AGG, pub));
    }
  }
  // ---- local exclusive scan of the tile counts over digits ----
  uint32_t inc = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm.wsum[warp] = inc;
  __syncthreads();
  uint32_t pre = 0;
#pragma unroll
  for (int w = 0; w < WARPS; ++w)
    if (w < warp) pre += (uint32_t)sm.wsum[w];
  uint32_t binst[BPT];
  {
    uint32_t run = pre + inc - tsum;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      binst[j] = run;
      if (own) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) sm.whist[w][tid * BPT + j] += run;   // fold the tile-local start
      }
      run += cnt[j];
    }
  }
  __syncthreads();

  // ---- scatter keys (and values) into shared memory in local digit order (frees registers) ----
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t d = dr[i] & 0xFFFFu;
    const uint32_t pos = sm.whist[warp][d] + (dr[i] >> 16);
    if (pos < (uint32_t)nvalid) {
      skeys[pos] = key[i];
      if (PAYLOAD || SRC == 2) svals[pos] = val[i];
    }
  }

  // ---- windowed decoupled look-back, publish the inclusive prefix, global digit offsets ----
  uint64_t excl[BPT];
#pragma unroll
  for (int j = 0; j < BPT; ++j) excl[j] = 0;
  if (tile > 0 && own) {
    if (EARLY)
      lookback_finish<BPT, W>(pa.status, BINS, tile, tid * BPT, pa.epoch, lbw, excl);
    else
      lookback_bins<BPT, W>(pa.status, BINS, tile, tid * BPT, pa.epoch, excl);
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const int b = tid * BPT + j;
      const uint32_t mine = (b == BINS - 1) ? cnt[j] - (uint32_t)(TILE - nvalid) : cnt[j];
      st_relaxed_u64(pa.status + (size_t)tile * BINS + b, st_pack(pa.epoch, ST_INC, excl[j] + mine));
    }
  }
#pragma unroll
  for (int j = 0; j < BPT; ++j)
    if (own) sm.gofs[tid * BPT + j] = pa.bases[tid * BPT + j] + excl[j] - binst[j];
  __syncthreads();

  // ---- write out: consecutive local slots of a digit go to consecutive global slots ----
  KeyT* kout = reinterpret_cast<KeyT*>(pa.keys_out);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int li = j * THREADS + tid;
    if (li < nvalid) {
      const KeyT k = skeys[li];
      const uint32_t dg = digit_of<KeyT, OWNER>(k, pa.pd, BINS - 1);
      const uint64_t g = sm.gofs[dg] + li;
      if constexpr (P2P) {
        static_assert((SRC == 3 || SRC == 0) && OWNER, "P2P is the dist bucketing pass");
        constexpr int K = Elem<T>::K;
        const uint64_t r = g - pa.bases[dg];   // rank inside the bucket of owner dg
        uint64_t* dd = pa.dst[dg];
        if (dd) dd[r] = (uint64_t)k;           // (a null destination drops the bucket: the own one,
        if ((int)dg != pa.self && dd) {        //  when the owner reads its incidences from conn)
          const int64_t e = (int64_t)((uint64_t)k & 0xffffffffull) - pa.elem_base;
          int row[K];
          load_row<T, false>(pa.conn, e, row);
          int32_t* rd = pa.rowdst[dg] + r * K;
#pragma unroll
          for (int q = 0; q < K; ++q) rd[q] = row[q];
        }
        continue;
      }
      if (!COUNTS) kout[g] = k;
      if (PAYLOAD || SRC == 2) pa.vals_out[g] = svals[li];
      if (COUNTS) {
        if (li == 0 || skeys[li - 1] != k) atomicAdd(pa.counts + k, -li);
        if (li == nvalid - 1 || skeys[li + 1] != k) atomicAdd(pa.counts + k, li + 1);
      }
    }
  }
}

// ================================================================================================
// k_unique_node: rows a4 + a5 fused for node mode.  Sorted keys in, warp-striped tiles:
//   flag(i)   = i == 0 || key[i] != key[i-1]                       (adjacent-difference dedupe)
//   pos(i)    = number of flags before i  (ballot/popc in the warp, look-back across tiles)
//   indices[pos(i)] = key[i] & (2^b - 1)  for flagged i             (compaction)
//   at a node change, offsets[x] = pos(i) for every node x in (node(key[i-1]), node(key[i])]
//   the last key fills offsets[x] = nnz for x in (node(last), N]     (run length + scan fused)
// ================================================================================================
struct UniqueArgs {
  const void* keys;
  int64_t n;
  int b;
  int64_t N;
  int64_t* offsets;
  uint32_t* indices;
  uint64_t* status;   // [tiles]
  uint32_t* ticket;
  uint32_t epoch;
  unsigned long long* nnz;
  const unsigned long long* err;
};

template <typename KeyT, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS, 3)
k_unique_node(UniqueArgs ua) {
  constexpr int WARPS = THREADS / 32;
  constexpr int TILE = THREADS * ITEMS;
  __shared__ uint32_t s_wcount[WARPS];
  __shared__ uint64_t s_texcl;
  __shared__ uint32_t s_tile;
  if (*ua.err != ERR_NONE) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ua.ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t chunk = (int64_t)tile * TILE + (int64_t)warp * 32 * ITEMS;
  const KeyT* keys = reinterpret_cast<const KeyT*>(ua.keys);

  KeyT key[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = chunk + i * 32 + lane;
    key[i] = idx < ua.n ? ld_stream(keys + idx) : (KeyT)0;
  }
  KeyT before = (KeyT)0;   // the key preceding this warp's chunk
  if (lane == 0 && chunk > 0 && chunk < ua.n) before = keys[chunk - 1];
  before = __shfl_sync(FULL, before, 0);

  // predecessor of item i in this lane (lane 0 takes lane 31 of item i-1, or `before`)
  auto prev_of = [&](int i) -> KeyT {
    const KeyT up = __shfl_up_sync(FULL, key[i], 1);
    const KeyT last = __shfl_sync(FULL, i > 0 ? key[i > 0 ? i - 1 : 0] : before, 31);
    return lane > 0 ? up : (i > 0 ? last : before);
  };

  unsigned bal[ITEMS];
  uint32_t wcount = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = chunk + i * 32 + lane;
    const KeyT p = prev_of(i);
    const bool f = idx < ua.n && (idx == 0 || key[i] != p);
    bal[i] = __ballot_sync(FULL, f);
    wcount += __popc(bal[i]);
  }
  if (lane == 0) s_wcount[warp] = wcount;
  __syncthreads();
  if (warp == 0) {
    uint32_t c = lane < WARPS ? s_wcount[lane] : 0;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    if (lane < WARPS) s_wcount[lane] = incl - c;
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed_u64(ua.status, st_pack(ua.epoch, ST_INC, tot));
    } else {
      if (lane == 0) st_relaxed_u64(ua.status + tile, st_pack(ua.epoch, ST_AGG, tot));
      excl = warp_lookback(ua.status, tile, ua.epoch, lane);
      if (lane == 0) st_relaxed_u64(ua.status + tile, st_pack(ua.epoch, ST_INC, excl + tot));
    }
    if (lane == 0) s_texcl = excl;
  }
  __syncthreads();
  uint64_t pos = s_texcl + s_wcount[warp];
  const KeyT vmask = (KeyT)(((KeyT)1 << ua.b) - 1);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = chunk + i * 32 + lane;
    const bool f = (bal[i] >> lane) & 1u;
    const uint64_t mypos = pos + __popc(bal[i] & lanemask_lt());
    const KeyT p = prev_of(i);
    if (f) {
      ua.indices[mypos] = (uint32_t)(key[i] & vmask);
      const int64_t a = (int64_t)(key[i] >> ua.b);
      const int64_t pa = idx == 0 ? -1 : (int64_t)(p >> ua.b);
      for (int64_t x = pa + 1; x <= a; ++x) ua.offsets[x] = (int64_t)mypos;
    }
    if (idx == ua.n - 1) {
      const uint64_t total = mypos + (f ? 1 : 0);
      for (int64_t x = (int64_t)(key[i] >> ua.b) + 1; x <= ua.N; ++x) ua.offsets[x] = (int64_t)total;
      *ua.nnz = total;
    }
    pos += __popc(bal[i]);
  }
}

// ================================================================================================
// Node neighbours from the element CSR (B200 restructure of rows a1/a3n/a4, DESIGN.md §"Node path").
// The paper's node pairs sorted by their first node are exactly the expansion of the element CSR:
// incidence (a, e) at element-CSR position i yields the C edge-neighbours of a inside e, so the
// pairs of node a are {nbr_p(conn[e]) : e in inc(a)} and only a per-node sort + adjacent-difference
// dedupe remains (segments of C*deg(a) entries: 12 tri, 72 Kuhn tet, 24 hex).  One thread per
// node (k_node_gather_t): private shared-memory hash set, insertion sort of the <= kMaxUnique
// distinct values, lists packed per CTA chunk; nodes with more distinct neighbours are queued for
// k_node_giant (block sort).  (A warp-per-node variant was 4x slower on B200 and was removed.)
// ================================================================================================
__device__ __forceinline__ uint32_t bitonic32(uint32_t x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(FULL, x, j);
      const bool asc = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      x = (lower == asc) ? min(x, y) : max(x, y);
    }
  }
  return x;
}

// Insert v into a per-warp open-addressing set tagged with the node (entry = tag | v).  Entries
// with another tag are free.  Returns true if v was not yet present for this node.
__device__ __forceinline__ bool hash_insert(unsigned long long* tab, unsigned long long tag, uint32_t v) {
  uint32_t h = (v * 0x9E3779B1u) >> 25;   // 128 slots
  const unsigned long long want = tag | v;
  for (int probe = 0; probe < 512; ++probe) {
    const unsigned long long cur = *(volatile unsigned long long*)(tab + h);
    if ((cur & 0xFFFFFFFF00000000ull) == tag) {
      if ((uint32_t)cur == v) return false;
      h = (h + 1) & 127;
      continue;
    }
    if (atomicCAS(tab + h, cur, want) == cur) return true;
  }
  return false;
}

template <int T, bool ALIGNED, bool RAND>
__device__ __forceinline__ void load_row(const int32_t* __restrict__ conn, int64_t e, int (&row)[Elem<T>::K]) {
  constexpr int K = Elem<T>::K;
  if (ALIGNED && (K == 4 || K == 8)) {
    const int4* p = reinterpret_cast<const int4*>(conn + e * K);
#pragma unroll
    for (int q = 0; q < K / 4; ++q) {
      const int4 x = RAND ? ldg_l2_64(p + q) : __ldg(p + q);
      row[4 * q] = x.x; row[4 * q + 1] = x.y; row[4 * q + 2] = x.z; row[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < K; ++q) row[q] = __ldg(conn + e * K + q);
  }
}

// Where element rows come from: the whole connectivity (1 GPU: base 0, M = all elements), or for
// a multi-GPU owner its own shard [base, base + M) plus a table of received remote rows whose
// element ids `relems` ascend (binary search).
struct RowSrc {
  const int32_t* conn;
  int64_t base, M;
  const int32_t* relems;
  const int32_t* rrows;
  int64_t nr;
};

template <int T, bool ALIGNED, bool DIST, bool RAND = false>
__device__ __forceinline__ void fetch_row(const RowSrc& rs, int64_t e, int (&row)[Elem<T>::K]) {
  if (!DIST) {   // 0 <= e < 2^31: 32-bit index, one wide multiply-add for the row address
    load_row<T, ALIGNED, RAND>(rs.conn, (uint64_t)(uint32_t)e, row);
    return;
  }
  if (e >= rs.base && e < rs.base + rs.M) {
    load_row<T, ALIGNED>(rs.conn, e - rs.base, row);
    return;
  }
  int64_t lo = 0, hi = rs.nr - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)rs.relems[mid] < e) lo = mid + 1; else hi = mid;
  }
  load_row<T, ALIGNED>(rs.rrows, lo, row);
}

template <int T>
__device__ __forceinline__ int local_of(const int (&row)[Elem<T>::K], int a) {
  int p = 0;
#pragma unroll
  for (int q = 0; q < Elem<T>::K; ++q) p = (row[q] == a) ? q : p;
  return p;
}

template <int T>
__device__ __forceinline__ uint32_t pick(const int (&row)[Elem<T>::K], int idx) {
  uint32_t v = 0;
#pragma unroll
  for (int q = 0; q < Elem<T>::K; ++q) v = (q == idx) ? (uint32_t)row[q] : v;
  return v;
}

constexpr int kSegThreads = 128;
constexpr int kSegMax = 32;   // longer element lists are sorted by k_segsort_giant

constexpr int next_pow2(int n) { return n <= 1 ? 1 : 2 * next_pow2((n + 1) / 2); }

// Batcher's odd-even merge sort on NET registers (ascending; NET need not be a power of two).
// The network for P = next_pow2(NET) inputs has only "min to the lower index" comparators, so
// +inf padding at positions >= NET stays there and every comparator touching those positions is a
// no-op: dropping them sorts NET values (24: 123 comparators vs 191 for 32; 32 vs bitonic: 191 vs
// 240).  Every index is a compile-time constant after unrolling, so v[] stays in registers.
struct CmpNet {
  int n;
  unsigned char a[256], b[256];
};
template <int NET>
constexpr CmpNet make_oem() {
  CmpNet t{};
  constexpr int P = next_pow2(NET);
  for (int p = 1; p < P; p <<= 1)
    for (int k = p; k >= 1; k >>= 1)
      for (int j = k % p; j + k < P; j += 2 * k)
        for (int i = 0; i < k; ++i) {
          const int a = i + j, b = i + j + k;
          if (b < NET && a / (2 * p) == b / (2 * p)) {
            t.a[t.n] = (unsigned char)a;
            t.b[t.n] = (unsigned char)b;
            ++t.n;
          }
        }
  return t;
}

template <int NET>
__device__ __forceinline__ void oddeven_sort(int32_t (&v)[NET]) {
  constexpr CmpNet T = make_oem<NET>();
  static_assert(T.n <= 256, "network too large");
#pragma unroll
  for (int c = 0; c < T.n; ++c) {
    const int32_t x = v[T.a[c]], y = v[T.b[c]];
    v[T.a[c]] = min(x, y);
    v[T.b[c]] = max(x, y);
  }
}

template <int NET>
__device__ __forceinline__ void sort_segment(int32_t* seg, int d) {
  int32_t v[NET];
#pragma unroll
  for (int i = 0; i < NET; ++i) v[i] = i < d ? seg[i] : INT32_MAX;
  oddeven_sort<NET>(v);
#pragma unroll
  for (int i = 0; i < NET; ++i)
    if (i < d) seg[i] = v[i];
}

// Thread-per-node variant (the one the pipeline uses): each thread walks its node's incidences
// (batched 4 at a time so the element-row gathers overlap), inserts the C neighbours of every
// incidence into a private open-addressing set in shared memory (column-major, so the 32 lanes of
// a warp always hit 32 different banks), insertion-sorts the <= kMaxUnique distinct values and
// writes them to the node's raw region.  Nodes with more distinct neighbours go to k_node_giant.
constexpr int kNodeThreads = 128;
constexpr int kHashSlots = 32;
constexpr int kMaxUnique = 24;

// The L <= NET distinct values in slots [0, L) of a thread's set column, sorted in registers and
// written to out[0, L).  Node ids are < 2^31, so INT32_MAX pads the network.
template <int NET, int HS>
__device__ __forceinline__ void sort_small(uint32_t (*tab)[kNodeThreads], int t, int L, uint32_t* out) {
  int32_t v[NET];
#pragma unroll
  for (int i = 0; i < NET; ++i) v[i] = (i < L && i < HS) ? (int32_t)tab[i < HS ? i : 0][t] : INT32_MAX;
  oddeven_sort<NET>(v);
#pragma unroll
  for (int i = 0; i < NET; ++i)
    if (i < L) out[i] = (uint32_t)v[i];
}

// The L <= NET values in the occupied slots of a thread's set column (bit i of `used` = slot i),
// read in slot order into registers (no compaction pass), sorted, written to out[0, L).
template <int NET>
__device__ __forceinline__ void sort_small_mask(uint32_t (*tab)[kNodeThreads], int t, uint32_t used, int L,
                                                uint32_t* out) {
  int32_t v[NET];
#pragma unroll
  for (int i = 0; i < NET; ++i) {
    const int slot = __ffs((int)used) - 1;   // (-1 once the mask is empty: not read then)
    used &= used - 1;
    v[i] = i < L ? (int32_t)tab[slot < 0 ? 0 : slot][t] : INT32_MAX;
  }
  oddeven_sort<NET>(v);
#pragma unroll
  for (int i = 0; i < NET; ++i)
    if (i < L) out[i] = (uint32_t)v[i];
}

// (Fusing the element-list sort of the transpose path into this kernel, with the CTA's incidence
// range staged in shared memory, was measured slower on B200: the extra registers / shared memory
// cost more occupancy than the saved pass.)
// SHARED: element-sharing ("FEM sparsity") adjacency — every other node of an incident element
// is a neighbour, so each incidence yields CE = K - 1 candidates.
// (prefetching the next batch's incidence window one batch ahead: 4.47 / 4.54 ms at 10 / 8 CTAs per
// SM vs 4.19 on config 5 -- not kept)
// >= 10 CTAs per SM (<= 48 registers) for arity <= 4: 4.48 vs 4.75 ms on config 5; hex keeps its
// registers for the 8-int rows (48 registers: 3.25 vs 2.63 ms on config 4).  profiles/round1/sweep_gather_minb.txt
// (Round 2 measured two attempts at a shorter probe chain slower and removed them: every candidate
// of a 4-incidence batch loading its home slot before any insert, 5.07 vs 4.13 ms on config 5; a
// per-batch instead of per-candidate set-capacity check with scalar incidence loads, 4.33-4.44 ms.
// DESIGN.md §5.)
template <int T, bool ALIGNED, bool DIST = false, bool SHARED = false, bool RAND = false,
          int MINB = (Elem<T>::K <= 4) ? 10 : 1>
__global__ void __launch_bounds__(kNodeThreads, MINB)
k_node_gather_t(const int64_t* __restrict__ eoff, const int32_t* __restrict__ eidx, RowSrc rs,
                int64_t N, uint32_t* __restrict__ temp, int32_t* __restrict__ cnt, int32_t* __restrict__ lofs,
                uint32_t* __restrict__ giants, unsigned int* __restrict__ ngiant,
                const unsigned long long* __restrict__ err, int64_t a_base = 0,
                int32_t* __restrict__ csum = nullptr) {
  constexpr int K = Elem<T>::K, B = 4;                   // incidences in flight per thread
  constexpr int C = SHARED ? K - 1 : Elem<T>::C;          // candidates per incidence
  constexpr uint32_t EMPTY = 0xFFFFFFFFu;
  // shared hex has 26 distinct neighbours per interior node: a 64-slot set, up to 40 kept; every
  // other instantiation 32 slots / 24 kept.  The distinct values are compacted in place at the end
  // (no separate list array: 16 KB / 32 KB per CTA, so registers, not shared memory, bound occupancy)
  constexpr bool WIDE = SHARED && K == 8;
  constexpr int HB = WIDE ? 6 : 5, HS = 1 << HB, MU = WIDE ? 40 : kMaxUnique;
  using Mask = typename std::conditional<(HS > 32), unsigned long long, uint32_t>::type;
  __shared__ uint32_t tab[HS][kNodeThreads];
  __shared__ uint32_t s_wsum[kNodeThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * kNodeThreads;
  const int64_t a = n0 + t;
  const bool valid = a < N;
  // the validation word and the node's offsets are loaded together (one latency, not two)
  const unsigned long long ev = err ? *err : ERR_NONE;
  const int64_t s0 = valid ? eoff[a] : 0;
  const int64_t d0 = valid ? eoff[a + 1] - s0 : 0;
  if (ev != ERR_NONE) return;
  const int32_t* inc = eidx + s0;
  int L = 0;
  int64_t raw = 0;
  Mask used = 0;   // occupied slots of the set
  if (valid) {
#pragma unroll
    for (int i = 0; i < HS; ++i) tab[i][t] = EMPTY;
    const int64_t d = d0;
    raw = (int64_t)C * d;
    for (int64_t i0 = 0; i0 < d && L <= MU; i0 += B) {
      // the B incidences from one or two aligned 16-byte loads (half the L1 lookups of B scalar
      // loads; the element CSR allocations carry 16 bytes of padding for the window)
      int e[B];
      {
        const int n = d - i0 < B ? (int)(d - i0) : B;
        const uintptr_t ad = reinterpret_cast<uintptr_t>(inc + i0);
        const int r = (int)((ad >> 2) & 3);
        const int4* ap = reinterpret_cast<const int4*>(ad & ~(uintptr_t)15);
        const int4 lo = __ldg(ap);
        const int4 hi = r + n > 4 ? __ldg(ap + 1) : lo;
        // e[q] = word q + r of the 8-word window: a two-level select on the bits of r (10 selects,
        // no divergent branches on the lane-dependent r)
        const bool r1 = (r & 2) != 0, r0 = (r & 1) != 0;
        const int u[5] = {r1 ? lo.z : lo.x, r1 ? lo.w : lo.y, r1 ? hi.x : lo.z, r1 ? hi.y : lo.w,
                          r1 ? hi.z : hi.x};
        // past the node's last incidence (n < B, a tail batch) the first incidence is repeated: its
        // candidates are already in the set, so the repeat only hits, and no incidence is skipped
        // by a branch (config 5's 24-incidence nodes have no tail batch)
#pragma unroll
        for (int q = 0; q < B; ++q) e[q] = r0 ? u[q + 1] : u[q];
#pragma unroll
        for (int q = 1; q < B; ++q) e[q] = q < n ? e[q] : e[0];
      }
      int row[B][K];
#pragma unroll
      for (int q = 0; q < B; ++q) fetch_row<T, ALIGNED, DIST, RAND>(rs, e[q], row[q]);
#pragma unroll
      for (int q = 0; q < B; ++q) {
        // simplices (TRI3, TET4): every other node of the element is an edge neighbour, so the
        // candidates are the row values != a; otherwise the local neighbour table is used
        constexpr bool simplex = (C == K - 1);   // simplices and SHARED: all other row values
        const int p = simplex ? 0 : local_of<T>(row[q], (int)(a + a_base));
        // simplex: the K - 1 values != a compacted with selects (other[j] = row[j + 1] once a has
        // been passed), so every lane inserts on every step (no divergent skip of a itself)
        uint32_t other[K > 1 ? K - 1 : 1];
        if (simplex) {
          bool passed = false;
#pragma unroll
          for (int j = 0; j < K - 1; ++j) {
            passed = passed || row[q][j] == (int)(a + a_base);
            other[j] = (uint32_t)(passed ? row[q][j + 1] : row[q][j]);
          }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const uint32_t v = simplex ? other[c] : pick<T>(row[q], nbr_local<T>(p, c));
          uint32_t h = (v * 0x9E3779B1u) >> (32 - HB);
          if (WIDE) {   // (measured: this form is 5% faster for the 64-slot set, 8% slower for 32)
            if (L <= MU) {   // at most MU + 1 entries: the set never fills
              // first probe resolves most candidates (hit or empty slot) without a branch
              uint32_t x = tab[h][t];
              if (x != v && x != EMPTY) {
                do {
                  h = (h + 1) & (HS - 1);
                  x = tab[h][t];
                } while (x != v && x != EMPTY);
              }
              if (x == EMPTY) {
                tab[h][t] = v;
                used |= Mask(1) << h;
                ++L;
              }
            }
          } else {
            while (L <= MU) {   // at most MU + 1 entries: the set never fills
              const uint32_t x = tab[h][t];
              if (x == v) break;
              if (x == EMPTY) {
                tab[h][t] = v;
                used |= Mask(1) << h;
                ++L;
                break;
              }
              h = (h + 1) & (HS - 1);
            }
          }
        }
      }
    }
  }
  const bool giant = valid && L > MU;
  // ---- dense per-CTA layout: node lists packed from C * eoff[n0]; a giant reserves raw slots ----
  const uint32_t size = valid ? (giant ? (uint32_t)raw : (uint32_t)L) : 0u;
  uint32_t incl = size;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t excl = incl - size;
#pragma unroll
  for (int w = 0; w < kNodeThreads / 32; ++w)
    if (w < warp) excl += s_wsum[w];
  if (csum && t == 0) {   // the chunk's list total (giants counted raw; k_node_giant corrects them)
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kNodeThreads / 32; ++w) tot += s_wsum[w];
    csum[blockIdx.x] = (int32_t)tot;
  }
  if (!valid) return;
  lofs[a] = (int32_t)excl;
  if (giant) {
    giants[atomicAdd(ngiant, 1u)] = (uint32_t)a;
    return;
  }
  if (!WIDE) {   // (L <= kMaxUnique = 24): the values go straight from the occupied slots (the mask)
    uint32_t* out = temp + (size_t)C * eoff[n0] + excl;
    const int lmax = __reduce_max_sync(__activemask(), (unsigned)L);
    if (lmax <= 8) sort_small_mask<8>(tab, t, (uint32_t)used, L, out);
    else if (lmax <= 16) sort_small_mask<16>(tab, t, (uint32_t)used, L, out);
    else sort_small_mask<24>(tab, t, (uint32_t)used, L, out);
    cnt[a] = L;
    return;
  }
  {   // compact the set to its first L slots (write index <= read index)
    int w = 0;
    while (used) {
      const int i = (HS > 32) ? __ffsll((long long)used) - 1 : __ffs((int)used) - 1;
      used &= used - 1;
      tab[w++][t] = tab[i][t];
    }
  }
  uint32_t* out = temp + (size_t)C * eoff[n0] + excl;
  // sort: a register bitonic network sized by the warp's largest set (warp-uniform, no divergence)
  const int lmax = __reduce_max_sync(__activemask(), (unsigned)L);
  if (lmax <= 8) sort_small<8, HS>(tab, t, L, out);
  else if (lmax <= 16) sort_small<16, HS>(tab, t, L, out);
  else if (lmax <= 24) sort_small<24, HS>(tab, t, L, out);
  else if (lmax <= 32) sort_small<32, HS>(tab, t, L, out);
  else {
    for (int i = 1; i < L; ++i) {
      const uint32_t x = tab[i][t];
      int j = i - 1;
      while (j >= 0 && tab[j][t] > x) {
        tab[j + 1][t] = tab[j][t];
        --j;
      }
      tab[j + 1][t] = x;
    }
    for (int i = 0; i < L; ++i) out[i] = tab[i][t];
  }
  cnt[a] = L;
}

// Block-wide: ascending bitonic sort of buf[0, raw) (implicit +inf padding to a power of two;
// pairs past raw are skipped), then the distinct values are written to out (in parallel: per-thread
// ranges + a block scan; serially by thread 0 when out aliases buf).  blockDim: a multiple of 32.
// Returns the distinct count (valid in every thread after the trailing barrier).
__device__ __forceinline__ int block_sort_dedupe(uint32_t* buf, int64_t raw, uint32_t* out) {
  __shared__ int s_u;
  int64_t n2 = 1;
  while (n2 < raw) n2 <<= 1;
  for (int64_t k = 2; k <= n2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
        int64_t lo, hi;
        const int64_t blk = t / j, o = t % j;
        if (j == (k >> 1)) {   // flip step: compare i with its mirror inside the k-block
          lo = blk * k + o;
          hi = blk * k + k - 1 - o;
        } else {
          lo = blk * 2 * j + o;
          hi = lo + j;
        }
        if (hi < raw) {
          const uint32_t x = buf[lo], y = buf[hi];
          if (x > y) { buf[lo] = y; buf[hi] = x; }
        }
      }
      __syncthreads();
    }
  }
  if (buf == out) {   // in place (global memory, > smem capacity): serial, reads ahead of writes
    if (threadIdx.x == 0) {
      int u = 0;
      for (int64_t i = 0; i < raw; ++i)
        if (i == 0 || buf[i] != buf[i - 1]) out[u++] = buf[i];
      s_u = u;
    }
    __syncthreads();
    return s_u;
  }
  // parallel: each thread a contiguous range, block exclusive scan of the distinct counts
  __shared__ int s_ws[32];
  const int nt = blockDim.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t per = (raw + nt - 1) / nt;
  const int64_t lo = (int64_t)t * per, hi = lo + per < raw ? lo + per : raw;
  int c = 0;
  for (int64_t i = lo; i < hi; ++i) c += (i == 0 || buf[i] != buf[i - 1]) ? 1 : 0;
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = nt >> 5;
    int x = lane < nw ? s_ws[lane] : 0, xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < nw) s_ws[lane] = xi - x;
    if (lane == nw - 1) s_u = xi;
  }
  __syncthreads();
  int pos = s_ws[warp] + incl - c;
  for (int64_t i = lo; i < hi; ++i)
    if (i == 0 || buf[i] != buf[i - 1]) out[pos++] = buf[i];
  __syncthreads();
  return s_u;
}

// Nodes with more than 256 raw neighbour entries (or more than 32 distinct neighbours): one CTA per
// node, the raw entries sorted with a block bitonic network (shared memory when they fit, else in
// place in the node's global raw region), then adjacent-difference dedupe.
template <int T, bool ALIGNED, bool DIST = false, bool SHARED = false>
__global__ void __launch_bounds__(1024)
k_node_giant(const int64_t* __restrict__ eoff, const int32_t* __restrict__ eidx, RowSrc rs,
             uint32_t* __restrict__ temp, int32_t* __restrict__ cnt, const int32_t* __restrict__ lofs,
             const uint32_t* __restrict__ giants, const unsigned int* __restrict__ ngiant, int smem_cap,
             const unsigned long long* __restrict__ err, int64_t a_base = 0, int32_t* __restrict__ csum = nullptr) {
  constexpr int K = Elem<T>::K;
  constexpr int C = SHARED ? K - 1 : Elem<T>::C;
  extern __shared__ uint32_t sv[];
  if (err && *err != ERR_NONE) return;
  const unsigned ng = *ngiant;
  for (unsigned g = blockIdx.x; g < ng; g += gridDim.x) {
    const int64_t a = giants[g];
    const int64_t s = eoff[a];
    const int64_t d = eoff[a + 1] - s;
    const int64_t raw = (int64_t)C * d;
    // the slot reserved by k_node_gather_t: raw entries at chunk base + lofs[a]
    uint32_t* out = temp + (size_t)C * eoff[(a / kNodeThreads) * kNodeThreads] + lofs[a];
    uint32_t* buf = raw <= smem_cap ? sv : out;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
      int row[K];
      fetch_row<T, ALIGNED, DIST>(rs, eidx[s + i], row);
      if (C == K - 1) {   // simplices and SHARED: the other row values
        int c = 0;
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (row[q] != (int)(a + a_base)) buf[i * C + (c++)] = (uint32_t)row[q];
      } else {
        const int p = local_of<T>(row, (int)(a + a_base));
#pragma unroll
        for (int c = 0; c < C; ++c) buf[i * C + c] = pick<T>(row, nbr_local<T>(p, c));
      }
    }
    __syncthreads();
    const int u = block_sort_dedupe(buf, raw, out);
    if (threadIdx.x == 0) {
      cnt[a] = u;
      if (csum) atomicAdd(csum + a / kNodeThreads, u - (int)raw);   // the chunk total held it raw
    }
    __syncthreads();
  }
}

// Node CSR indices: a CTA per kNodeThreads-node chunk (the same chunks as k_node_gather_t, whose
// lists are packed from C * eoff[n0]) writes its contiguous output range with consecutive threads
// on consecutive positions; the node of each position is found by binary search in shared memory.
__global__ void __launch_bounds__(kNodeThreads)
k_node_compact(const int64_t* __restrict__ eoff, int C, const uint32_t* __restrict__ temp,
               const int32_t* __restrict__ lofs, const int64_t* __restrict__ noff, int64_t N,
               int32_t* __restrict__ out, const int64_t* __restrict__ rawoff = nullptr) {
  __shared__ int64_t s_src[kNodeThreads];
  __shared__ int64_t s_dst[kNodeThreads + 1];
  const int64_t n0 = (int64_t)blockIdx.x * kNodeThreads;
  const int t = threadIdx.x;
  const int nloc = (int)(N - n0 < kNodeThreads ? N - n0 : kNodeThreads);
  const int64_t base = rawoff ? rawoff[n0] : (int64_t)C * eoff[n0];   // (rawoff: polygon meshes)
  if (t < nloc) {
    s_src[t] = base + lofs[n0 + t];
    s_dst[t] = noff[n0 + t];
  }
  if (t == 0) s_dst[nloc] = noff[n0 + nloc];
  __syncthreads();
  const int64_t o0 = s_dst[0], o1 = s_dst[nloc];
  // without a giant in the chunk the packed source layout equals the destination layout
  const bool packed = __syncthreads_and(t >= nloc || s_src[t] - base == s_dst[t] - o0);
  if (packed) {
    const uint32_t* src = temp + base - o0;
    for (int64_t o = o0 + t; o < o1; o += kNodeThreads) out[o] = (int32_t)src[o];
    return;
  }
  for (int64_t o = o0 + t; o < o1; o += kNodeThreads) {
    int lo = 0, hi = nloc - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_dst[mid] <= o) lo = mid; else hi = mid - 1;
    }
    out[o] = (int32_t)temp[s_src[lo] + (o - s_dst[lo])];
  }
}

// k_node_compact with the node-offset scan folded in: a chunk's base is cb[chunk] (the exclusive scan
// of the per-chunk list totals k_node_gather_t / k_node_giant leave in csum), each node's offset is
// that base + the CTA's exclusive scan of the node counts; writes offsets[n0 .. n0 + nloc) (and
// offsets[N] in the last chunk) and copies the lists (none when out == nullptr, i.e. nnz == 0).
// Replaces a look-back scan over the N counts (0.17 ms on config 5) by one over N / 128 totals.
__global__ void __launch_bounds__(kNodeThreads)
k_node_compact_cb(const int64_t* __restrict__ eoff, int C, const uint32_t* __restrict__ temp,
                  const int32_t* __restrict__ lofs, const int32_t* __restrict__ cnt, const int64_t* __restrict__ cb,
                  int64_t N, int64_t* __restrict__ noff, int32_t* __restrict__ out) {
  __shared__ int64_t s_src[kNodeThreads];
  __shared__ int64_t s_dst[kNodeThreads + 1];
  __shared__ int s_w[kNodeThreads / 32];
  const int64_t n0 = (int64_t)blockIdx.x * kNodeThreads;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nloc = (int)(N - n0 < kNodeThreads ? N - n0 : kNodeThreads);
  const int64_t base = (int64_t)C * eoff[n0];
  const int d = t < nloc ? cnt[n0 + t] : 0;
  int incl = d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int excl = incl - d;
#pragma unroll
  for (int w = 0; w < kNodeThreads / 32; ++w)
    if (w < warp) excl += s_w[w];
  const int64_t o = cb[blockIdx.x] + excl;
  if (t < nloc) {
    s_src[t] = base + lofs[n0 + t];
    s_dst[t] = o;
    noff[n0 + t] = o;
  }
  if (t == nloc - 1) {
    s_dst[nloc] = o + d;
    if (n0 + nloc == N) noff[N] = o + d;
  }
  __syncthreads();
  if (!out) return;
  const int64_t o0 = s_dst[0], o1 = s_dst[nloc];
  // without a giant in the chunk the packed source layout equals the destination layout
  const bool packed = __syncthreads_and(t >= nloc || s_src[t] - base == s_dst[t] - o0);
  if (packed) {
    const uint32_t* src = temp + base - o0;
    for (int64_t i = o0 + t; i < o1; i += kNodeThreads) out[i] = (int32_t)src[i];
    return;
  }
  for (int64_t i = o0 + t; i < o1; i += kNodeThreads) {
    int lo = 0, hi = nloc - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_dst[mid] <= i) lo = mid; else hi = mid - 1;
    }
    out[i] = (int32_t)temp[s_src[lo] + (i - s_dst[lo])];
  }
}

// ================================================================================================
// Element CSR as a counting-sort transpose, used when the mesh numbering has
// locality: the element CSR is the transpose of the incidence matrix B.
//   k_locality_sample  distinct (slot, node) groups per warp window of 32 consecutive elements
//                      (chooses the transpose; the transpose itself is the chunk-bucketed one below)
//   k_elem_segsort     per-node register sort of element-id segments (the polygon sharing path)
//   k_segsort_giant    block bitonic sort for segments longer than kSegMax
// (the per-node count / scatter kernels this path started with -- 7.1 ms on config 5 against
// 4.6 ms for the chunk buckets -- were removed once every mode moved to the chunk buckets)
// ================================================================================================
template <int T, bool ALIGNED>
__global__ void __launch_bounds__(256)
k_locality_sample(const int32_t* __restrict__ conn, int64_t M, unsigned long long* __restrict__ out) {
  constexpr int K = Elem<T>::K;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t e0 = (int64_t)((double)M * (double)gw / (double)nw);
  const int64_t e = e0 + lane;
  const bool in = e < M;
  int row[K];
  if (in) load_row<T, ALIGNED>(conn, e, row);
  unsigned groups = 0;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const int x = in ? row[p] : -1;   // one shared sentinel: match cost grows with distinct values
    const unsigned peers = __match_any_sync(FULL, x);
    groups += (in && lane == __ffs(peers) - 1) ? 1u : 0u;
  }
  const unsigned act = __popc(__ballot_sync(FULL, in));
  groups = __reduce_add_sync(FULL, groups);
  if (lane == 0) {
    atomicAdd(out, (unsigned long long)groups);
    atomicAdd(out + 1, (unsigned long long)act * K);
  }
}




constexpr int kSegSmem = 8192;   // elements of a 128-node chunk staged in shared memory

// A CTA per kSegThreads consecutive nodes: their segments form one contiguous range, staged
// through shared memory with coalesced loads/stores; each thread sorts its own segment with a
// register sorting network sized by the largest segment of its warp (warp-uniform choice).
template <int SMEM = kSegSmem, int MINB = 1>
__global__ void __launch_bounds__(kSegThreads, MINB)
k_elem_segsort(const int64_t* __restrict__ eoff, int64_t N, int32_t* __restrict__ eidx,
               uint32_t* __restrict__ giants, unsigned int* __restrict__ ngiant,
               const unsigned long long* __restrict__ err) {
  __shared__ int32_t buf[SMEM];
  if (err && *err != ERR_NONE) return;
  const int t = threadIdx.x;
  const int64_t n0 = (int64_t)blockIdx.x * kSegThreads;
  const int64_t n1 = n0 + kSegThreads < N ? n0 + kSegThreads : N;
  const int64_t c0 = eoff[n0], c1 = eoff[n1];
  const int64_t a = n0 + t;
  const bool valid = a < N;
  const int64_t s = valid ? eoff[a] : c1;
  const int d = valid ? (int)(eoff[a + 1] - s) : 0;
  const bool big = d > kSegMax;
  if (valid && big) giants[atomicAdd(ngiant, 1u)] = (uint32_t)a;
  const bool staged = c1 - c0 <= SMEM;   // CTA-uniform
  if (staged) {
    for (int64_t i = c0 + t; i < c1; i += kSegThreads) buf[i - c0] = eidx[i];
    __syncthreads();
  }
  int32_t* seg = staged ? buf + (s - c0) : eidx + s;
  const int dd = (valid && !big) ? d : 0;
  const int wmax = __reduce_max_sync(0xffffffffu, (unsigned)dd);
  if (wmax > 1) {
    if (wmax <= 8) sort_segment<8>(seg, dd);
    else if (wmax <= 16) sort_segment<16>(seg, dd);
    else if (wmax <= 24) sort_segment<24>(seg, dd);
    else sort_segment<32>(seg, dd);
  }
  if (staged) {
    __syncthreads();
    // giants keep their (unsorted) values here and are sorted by k_segsort_giant afterwards
    for (int64_t i = c0 + t; i < c1; i += kSegThreads) eidx[i] = buf[i - c0];
  }
}

// ------------------------------------------------------------------------------------------------
// Chunk-bucketed transpose (the default element path for meshes with locality).  The incidences
// are bucketed by 128-node chunk (one bucket per kChunkNodes consecutive nodes) instead of by node:
//   k_chunk_count    validation + per-chunk incidence counts, one atomic per (warp, slot, chunk)
//                    group (__match_any_sync; consecutive elements of a coherent mesh hit 1-3 chunks)
//   k_scan_i32       chunk bases
//   k_chunk_scatter  appends (element id, local node) to the chunk's bucket: runs of consecutive
//                    slots, so only a bucket's tail sector is ever partially written
//   k_chunk_sort     one CTA per chunk: bucket -> fixed per-node slots in shared memory, each
//                    node's list sorted in registers (warp-uniform network), element CSR range and
//                    the chunk's offsets written coalesced; lists > kSegMax go to k_segsort_giant
// ------------------------------------------------------------------------------------------------
#ifndef MN_CHUNK_SHIFT
#define MN_CHUNK_SHIFT 7
#endif
// log2 of the nodes per chunk (local node ids fit a byte).  256-node chunks (-DMN_CHUNK_SHIFT=8),
// config 5: scatter 2.12 vs 2.15 ms, chunk sort 2.53 vs 2.37 -> 128 kept
constexpr int kChunkShift = MN_CHUNK_SHIFT;
constexpr int kChunkNodes = 1 << kChunkShift;
static_assert(kChunkNodes <= 256, "local node ids are bytes");
constexpr int kChunkCap = 4096;   // bucket entries staged in shared memory (Kuhn tets: 3072)
constexpr int kStage = 3584;      // k_chunk_sort: bucket entries read by bulk copy (larger: register loads; 6 CTAs/SM)

// RANGE: only nodes of [lo, hi) (the memory-bounded mode); compiled out of the whole-path kernels
template <int T, bool ALIGNED, bool RANGE = false>
__global__ void __launch_bounds__(256)
k_chunk_count(const int32_t* __restrict__ conn, int64_t M, int64_t N, int32_t* __restrict__ ccnt,
              unsigned long long* __restrict__ err, int64_t lo = 0, int64_t hi = INT64_MAX,
              const unsigned int* __restrict__ guard = nullptr) {
  constexpr int K = Elem<T>::K;
  if (guard && *guard == 0u) return;   // fallback after a fixed-capacity bucket overflowed
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < M; base += stride) {
    const int64_t e = base + lane;
    const bool in = e < M;
    int v[K];
    if (in) load_row<T, ALIGNED>(conn, e, v);
    int kind = 0;
    const int bad = in ? row_bad<K>(v, (uint32_t)N, kind) : -1;
    if (in) {
      if (bad >= 0) atomicMin(err, (unsigned long long)err_encode((uint64_t)e, kind, bad));
    }
    const bool ok = in && bad < 0;
#pragma unroll
    for (int p = 0; p < K; ++p) {   // only nodes of [lo, hi) (the memory-bounded mode's range)
      const bool mine = ok && (!RANGE || (v[p] >= lo && v[p] < hi));
      const int x = mine ? (RANGE ? (int)((v[p] - lo) >> kChunkShift) : (v[p] >> kChunkShift)) : -1;   // one shared sentinel
      const unsigned peers = __match_any_sync(FULL, x);   // (match cost grows with distinct values)
      if (mine && lane == __ffs(peers) - 1) atomicAdd(ccnt + x, (int)__popc(peers));
    }
  }
}

template <int T, bool ALIGNED, bool RANGE = false>
__global__ void __launch_bounds__(256)
k_chunk_scatter(const int32_t* __restrict__ conn, int64_t M, const int64_t* __restrict__ cbase,
                int32_t* __restrict__ ccur, int32_t* __restrict__ belem, uint8_t* __restrict__ bnode,
                const unsigned long long* __restrict__ err, int64_t lo = 0, int64_t hi = INT64_MAX,
                const unsigned int* __restrict__ guard = nullptr, int64_t ebase = 0) {
  constexpr int K = Elem<T>::K;
  if (guard && *guard == 0u) return;   // fallback after a fixed-capacity bucket overflowed
  if (*err != ERR_NONE) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < M; base += stride) {
    const int64_t e = base + lane;
    const bool in = e < M;
    int v[K];
    if (in) load_row<T, ALIGNED>(conn, e, v);
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const bool mine = in && (!RANGE || (v[p] >= lo && v[p] < hi));
      const int x = mine ? (RANGE ? (int)((v[p] - lo) >> kChunkShift) : (v[p] >> kChunkShift)) : -1;   // one shared sentinel
      const unsigned peers = __match_any_sync(FULL, x);
      const int leader = __ffs(peers) - 1;
      int b = 0;
      if (mine && lane == leader) b = atomicAdd(ccur + x, (int)__popc(peers));
      b = __shfl_sync(FULL, b, leader);
      if (mine) {
        const int64_t pos = cbase[x] + b + __popc(peers & lanemask_lt());
        belem[pos] = (int32_t)(ebase + e);
        bnode[pos] = (uint8_t)((RANGE ? (int)(v[p] - lo) : v[p]) & (kChunkNodes - 1));
      }
    }
  }
}

// One warp-block (32 consecutive elements) of k_chunk_scatter_fixed between its two stages.
template <int K>
struct ScatterBlock {
  uint32_t e;
  int v[K], x[K], b[K];
  unsigned peers[K];
};

// Stage A: validation, chunk of every incidence, warp groups (__match_any_sync), and the leader's
// returning atomic on the chunk cursor (its result is consumed one block later, in stage B).
template <int K, bool RANGE>
__device__ __forceinline__ void scatter_stage_a(ScatterBlock<K>& s, uint32_t base, int lane, uint32_t end,
                                                const int (&row)[K], uint32_t N, int64_t lo, int64_t hi,
                                                int32_t* __restrict__ ccur, unsigned long long* __restrict__ err) {
  s.e = base + lane;
  const bool in = s.e < end;
#pragma unroll
  for (int p = 0; p < K; ++p) s.v[p] = row[p];
  int kind = 0;
  const int bad = in ? row_bad<K>(s.v, N, kind) : -1;
  if (in && bad >= 0) atomicMin(err, (unsigned long long)err_encode((uint64_t)s.e, kind, bad));
  const bool ok = in && bad < 0;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const bool mine = ok && (!RANGE || (s.v[p] >= lo && s.v[p] < hi));
    s.x[p] = mine ? (int)((RANGE ? s.v[p] - lo : s.v[p]) >> kChunkShift) : -1;   // one shared sentinel (match cost grows with distinct values)
    s.peers[p] = __match_any_sync(FULL, s.x[p]);
    s.b[p] = 0;
    if (s.x[p] >= 0 && lane == __ffs(s.peers[p]) - 1) s.b[p] = atomicAdd(ccur + s.x[p], (int)__popc(s.peers[p]));
  }
}

// Stage B: each incidence's slot = its leader's cursor value + its rank in the group; writes.
template <int K, bool RANGE>
__device__ __forceinline__ void scatter_stage_b(const ScatterBlock<K>& s, int lane, int cap, int64_t lo, int64_t ebase,
                                                int32_t* __restrict__ belem, uint8_t* __restrict__ bnode, bool& over) {
  const int32_t eid = (int32_t)(ebase + s.e);
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const int leader = __ffs(s.peers[p]) - 1;
    const int q = __shfl_sync(FULL, s.b[p], leader) + __popc(s.peers[p] & lanemask_lt());
    if (s.x[p] >= 0) {
      if (q < cap) {
        const uint64_t pos = (uint64_t)(uint32_t)s.x[p] * (uint32_t)cap + (uint32_t)q;   // one wide multiply-add
        belem[pos] = eid;
        bnode[pos] = (uint8_t)((RANGE ? s.v[p] - lo : s.v[p]) & (kChunkNodes - 1));
      } else {
        over = true;
      }
    }
  }
}

// Single-read variant for the whole-path call (no count pass): validation (as k_chunk_count) and
// the scatter into fixed-capacity buckets, chunk x at [x * cap, (x + 1) * cap).  The cursors end as
// the chunk counts; a scan of them gives the element-CSR chunk bases.  A chunk whose count exceeds
// cap sets *ovf and keeps only its first cap entries: the host queues the counted path
// (k_chunk_count -> k_scan_i32 -> k_chunk_scatter, each guarded by *ovf) behind it, so the result
// never depends on cap.  Saves the count pass's read of conn (config 5: 1.08 ms of 11.3).
// RANGE (multi-GPU owners): only nodes of [lo, hi) are kept (local ids node - lo) and element ids
// are written as ebase + e (the shard's global ids).
template <int T, bool ALIGNED, int MINB = 1, bool RANGE = false>
__global__ void __launch_bounds__(256, MINB)
k_chunk_scatter_fixed(const int32_t* __restrict__ conn, int64_t M, int64_t N, int cap,
                      int32_t* __restrict__ ccur, int32_t* __restrict__ belem, uint8_t* __restrict__ bnode,
                      unsigned long long* __restrict__ err, unsigned int* __restrict__ ovf, int64_t lo = 0,
                      int64_t hi = INT64_MAX, int64_t ebase = 0) {
  constexpr int K = Elem<T>::K;
  const int lane = threadIdx.x & 31;
  // (grid-stride; a blocked assignment, each CTA on its own contiguous element range so that few
  // CTAs share a chunk counter at a time, measured the same: 2.10-2.28 vs 2.14 ms on config 5)
  // 32-bit element indices (M <= INT32_MAX, checked at the C ABI; base + stride < 2^32).
  // Software-pipelined by one block: the returning cursor atomics of block i + 1 are issued before
  // the writes of block i wait on block i's (60% of the stall samples sat on those results, r2o).
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  const uint32_t end = (uint32_t)M;
  bool over = false;   // some incidence of this thread found its bucket full (flagged once at the end)
  if (base >= end) return;
  ScatterBlock<K> cur, nxt;
  int nv[K];   // the row of the block after the one in stage A, loaded one block ahead
  if (base + lane < end) load_row<T, ALIGNED>(conn, (uint64_t)(base + lane), nv);
  if (base + stride + lane < end) {
    int r[K];
    load_row<T, ALIGNED>(conn, (uint64_t)(base + stride + lane), r);
    scatter_stage_a<K, RANGE>(cur, base, lane, end, nv, (uint32_t)N, lo, hi, ccur, err);
#pragma unroll
    for (int p = 0; p < K; ++p) nv[p] = r[p];
  } else {
    scatter_stage_a<K, RANGE>(cur, base, lane, end, nv, (uint32_t)N, lo, hi, ccur, err);
  }
  for (; base < end; base += stride) {
    const uint32_t next = base + stride;
    if (next < end) {
      int r[K];
      const bool pre = next + stride + lane < end;
      if (pre) load_row<T, ALIGNED>(conn, (uint64_t)(next + stride + lane), r);
      scatter_stage_a<K, RANGE>(nxt, next, lane, end, nv, (uint32_t)N, lo, hi, ccur, err);
      if (pre) {
#pragma unroll
        for (int p = 0; p < K; ++p) nv[p] = r[p];
      }
    }
    scatter_stage_b<K, RANGE>(cur, lane, cap, lo, ebase, belem, bnode, over);
    cur = nxt;
  }
  if (over) *ovf = 1u;
}

// One CTA (kChunkNodes threads) per chunk, one pass over the bucket (SORT = false, node-only
// calls, groups by node without ordering each list).  Each local node owns kSegMax fixed slots (column t of a skewed
// 32 x 129 array: per-thread column reads and per-warp row copies are both conflict-free); the slot
// cursor is the count.  A node with more than kSegMax entries flags the chunk, which then takes the
// two-pass global path (counts already known).  Sorted lists go back to their columns and each warp
// copies its 32 nodes' lists out, one coalesced store per node.  (2.77 ms on config 5; measured
// slower: a count pass + skewed staging array, 3.11 ms; staging the bucket in shared memory, 3.43;
// warp-aggregating the shared atomics with __match_any_sync, 7.39; 8-entry vector groups, 3.65.)
constexpr int kSlotPitch = kChunkNodes + 1;

template <int NET>
__device__ __forceinline__ void sort_slot_column(int32_t* slots, int t, int d) {
  int32_t v[NET];
#pragma unroll
  for (int i = 0; i < NET; ++i) v[i] = i < d ? slots[i * kSlotPitch + t] : INT32_MAX;
  oddeven_sort<NET>(v);
#pragma unroll
  for (int i = 0; i < NET; ++i)
    if (i < d) slots[i * kSlotPitch + t] = v[i];
}

template <bool SORT, int MINB = 6>
__global__ void __launch_bounds__(kChunkNodes, MINB)
k_chunk_sort(const int64_t* __restrict__ cbase, int64_t N, const int32_t* __restrict__ belem,
              const uint8_t* __restrict__ bnode, int64_t* __restrict__ eoff, int32_t* __restrict__ eidx,
              uint32_t* __restrict__ giants, unsigned int* __restrict__ ngiant,
              const unsigned long long* __restrict__ err, const unsigned int* __restrict__ ovf = nullptr,
              int cap = 0) {
  __shared__ int32_t slots[kSegMax * kSlotPitch];
  __shared__ int s_cnt[kChunkNodes];
  __shared__ int s_ex[kChunkNodes];
  __shared__ int2 s_ce[kChunkNodes];   // (count, offset) per node for the copy-out (one 8-byte load)
  __shared__ int s_wsum[kChunkNodes / 32];
  __shared__ int s_over;
  __shared__ alignas(16) int32_t s_el[kStage];   // the bucket, brought in by two bulk copies
  __shared__ alignas(16) uint8_t s_nd[kStage];
  __shared__ alignas(8) uint64_t s_bar;
  if (err && *err != ERR_NONE) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t c = blockIdx.x;
  const int64_t n0 = c * kChunkNodes;
  const int64_t b0 = cbase[c], b1 = cbase[c + 1];
  const int n = (int)(b1 - b0);
  // where the bucket is: fixed-capacity layout (k_chunk_scatter_fixed) unless it overflowed
  const bool fixed = ovf && *ovf == 0u;
  const int64_t bb = fixed ? c * (int64_t)cap : b0;
  // CTA-uniform: a fixed-capacity bucket (cap a multiple of 16, so the copies rounded up to 16
  // entries stay inside it) that fits the stage is read with TMA bulk copies -- the whole bucket in
  // flight at once instead of one 4-entry group per thread (the register-load version waited on
  // its loads for 35% of its samples, ncu r1v)
  const bool bulk = fixed && (cap & 15) == 0 && n > 0 && n <= kStage;
  if (bulk && t == 0) mbar_init(&s_bar, 1);
  s_cnt[t] = 0;
  if (t == 0) s_over = 0;
  __syncthreads();
  constexpr int U = 4;
  if (bulk) {
    if (t == 0) {
      const uint32_t be = (uint32_t)((n + 3) & ~3) * 4u, bn = (uint32_t)((n + 15) & ~15);   // within cap
      mbar_arrive_expect_tx(&s_bar, be + bn);
      bulk_g2s(s_el, belem + bb, be, &s_bar);
      bulk_g2s(s_nd, bnode + bb, bn, &s_bar);
    }
    mbar_wait(&s_bar, 0);
    const int nfull = n & ~(U - 1);   // full 4-entry groups without per-entry bounds checks
    for (int i0 = 0; i0 < nfull; i0 += U * kChunkNodes) {
      const int i = i0 + U * t;
      if (i >= nfull) break;
      const uint32_t nq = *reinterpret_cast<const uint32_t*>(s_nd + i);
      const int4 eq = *reinterpret_cast<const int4*>(s_el + i);
      const int nd[U] = {(int)(nq & 255), (int)((nq >> 8) & 255), (int)((nq >> 16) & 255), (int)(nq >> 24)};
      const int32_t el[U] = {eq.x, eq.y, eq.z, eq.w};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int pos = atomicAdd(&s_cnt[nd[u]], 1);
        if (pos < kSegMax) slots[pos * kSlotPitch + nd[u]] = el[u];
        else s_over = 1;
      }
    }
    if (t < n - nfull) {   // the <= 3 entries of the last partial group
      const int i = nfull + t, nd = s_nd[i];
      const int pos = atomicAdd(&s_cnt[nd], 1);
      if (pos < kSegMax) slots[pos * kSlotPitch + nd] = s_el[i];
      else s_over = 1;
    }
  } else if ((bb & 15) == 0) {   // CTA-uniform: 16-byte aligned bucket (the fixed layout) -> vector loads
    // thread t takes entries [i0 + 4t, i0 + 4t + 4): one 4-byte node load + one int4 element load
    for (int i0 = 0; i0 < n; i0 += U * kChunkNodes) {
      const int i = i0 + U * t;
      int nd[U];
      int32_t el[U];
      if (i + U <= n) {
        const uint32_t nq = __ldg(reinterpret_cast<const uint32_t*>(bnode + bb + i));
        const int4 eq = __ldg(reinterpret_cast<const int4*>(belem + bb + i));
        nd[0] = nq & 255; nd[1] = (nq >> 8) & 255; nd[2] = (nq >> 16) & 255; nd[3] = nq >> 24;
        el[0] = eq.x; el[1] = eq.y; el[2] = eq.z; el[3] = eq.w;
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          nd[u] = i + u < n ? (int)__ldg(bnode + bb + i + u) : -1;
          el[u] = i + u < n ? __ldg(belem + bb + i + u) : 0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (nd[u] >= 0) {
          const int pos = atomicAdd(&s_cnt[nd[u]], 1);
          if (pos < kSegMax) slots[pos * kSlotPitch + nd[u]] = el[u];
          else s_over = 1;
        }
    }
  } else {
  for (int i0 = 0; i0 < n; i0 += U * kChunkNodes) {
    int nd[U];
    int32_t el[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kChunkNodes + t;
      nd[u] = i < n ? (int)__ldg(bnode + bb + i) : -1;
      el[u] = i < n ? __ldg(belem + bb + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (nd[u] >= 0) {
        const int pos = atomicAdd(&s_cnt[nd[u]], 1);
        if (pos < kSegMax) slots[pos * kSlotPitch + nd[u]] = el[u];
        else s_over = 1;
      }
  }
  }
  __syncthreads();
  const int d = s_cnt[t];
  int incl = d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int excl = incl - d;
#pragma unroll
  for (int w = 0; w < kChunkNodes / 32; ++w)
    if (w < warp) excl += s_wsum[w];
  const int64_t a = n0 + t;
  if (a < N) eoff[a] = b0 + excl;
  if (a == N - 1) eoff[N] = b1;
  s_ex[t] = excl;
  s_ce[t] = make_int2(d, excl);
  const bool over = s_over != 0;   // CTA-uniform (read after the barrier above)
  if (!over) {
    const int dd = SORT ? d : 0;
    const int wmax = __reduce_max_sync(FULL, (unsigned)dd);
    if (wmax > 1) {
      if (wmax <= 8) sort_slot_column<8>(slots, t, dd);
      else if (wmax <= 16) sort_slot_column<16>(slots, t, dd);
      else if (wmax <= 24) sort_slot_column<24>(slots, t, dd);
      else sort_slot_column<32>(slots, t, dd);
    }
    __syncthreads();
    if (n >= 8 * kChunkNodes) {   // (config 5, mean 24: 2.69 ms this way, 3.25 position-mapped)
      // long lists (mean >= 8): warp w copies the lists of nodes 32w .. 32w+31, lane i writing
      // entry i of the node (one coalesced store per node)
      int32_t* const ob = eidx + b0;   // (32-bit offsets inside the chunk's output range)
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        const int nodeq = warp * 32 + q;
        const int2 ce = s_ce[nodeq];
        if (lane < ce.x) ob[ce.y + lane] = slots[lane * kSlotPitch + nodeq];
      }
    } else {
      // short lists: thread i writes chunk output position i; its node by binary search in s_ex
      for (int i = t; i < n; i += kChunkNodes) {
        int lo = 0;
#pragma unroll
        for (int step = kChunkNodes / 2; step > 0; step >>= 1)
          if (s_ex[lo + step] <= i) lo += step;
        eidx[b0 + i] = slots[(i - s_ex[lo]) * kSlotPitch + lo];
      }
    }
    return;
  }
  // overflowed chunk: place in global memory with the known counts, sort there (lists > kSegMax
  // go to k_segsort_giant)
  __syncthreads();
  s_cnt[t] = excl;
  __syncthreads();
  for (int i = t; i < n; i += kChunkNodes) {
    const int slot = atomicAdd(&s_cnt[(int)__ldg(bnode + bb + i)], 1);
    eidx[b0 + slot] = __ldg(belem + bb + i);
  }
  const bool big = d > kSegMax;
  if (a < N && big && SORT) giants[atomicAdd(ngiant, 1u)] = (uint32_t)a;
  const int dd = (SORT && !big) ? d : 0;
  const int wmax = __reduce_max_sync(FULL, (unsigned)dd);
  __syncthreads();   // the CTA's global writes are visible to the CTA after the barrier
  if (wmax > 1) {
    int32_t* seg = eidx + b0 + excl;
    if (wmax <= 8) sort_segment<8>(seg, dd);
    else if (wmax <= 16) sort_segment<16>(seg, dd);
    else if (wmax <= 24) sort_segment<24>(seg, dd);
    else sort_segment<32>(seg, dd);
  }
}

// ------------------------------------------------------------------------------------------------
// MSD element path for meshes without locality: one onesweep pass buckets the
// (node, element) pairs stably by node range [g * R, (g + 1) * R) (owner digit node / R, 512
// buckets), then one CTA per bucket finishes the transpose in shared memory instead of the
// remaining LSD passes: per-node counts (shared atomics on R <= kRangeMax counters), block scan ->
// element-CSR offsets, scatter of the element ids into their node segments (the bucket's output
// range, L2-resident), and a register sort per segment (lists > kSegMax go to k_segsort_giant).
// ------------------------------------------------------------------------------------------------
constexpr int kRangeThreads = 1024;
constexpr int kRangeMax = 48 * 1024;   // nodes per bucket (192 KB of counters)

template <bool SORT>
__global__ void __launch_bounds__(kRangeThreads, 1)
k_range_transpose(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                  const uint64_t* __restrict__ bases, int nb, int R, int64_t N, int64_t total,
                  int64_t* __restrict__ eoff, int32_t* __restrict__ eidx, uint32_t* __restrict__ giants,
                  unsigned int* __restrict__ ngiant, const unsigned long long* __restrict__ err) {
  extern __shared__ int32_t scnt[];
  __shared__ int s_ws[kRangeThreads / 32];
  if (err && *err != ERR_NONE) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // persistent: a grid smaller than nb keeps the CTAs' random-write windows (one bucket's element
  // ids each) inside L2
  for (int g = blockIdx.x; g < nb; g += gridDim.x) {
  __syncthreads();
  const int64_t lo = (int64_t)g * R;
  if (lo >= N) continue;
  const int nr = (int)(lo + R < N ? R : N - lo);
  const int64_t b0 = (int64_t)bases[g], b1 = g + 1 < nb ? (int64_t)bases[g + 1] : total;
  for (int j = t; j < nr; j += kRangeThreads) scnt[j] = 0;
  __syncthreads();
  constexpr int U = 8;   // loads in flight per thread (each pass is otherwise one round trip per entry)
  for (int64_t i0 = b0 + t; i0 < b1; i0 += (int64_t)U * kRangeThreads) {
    uint32_t k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * kRangeThreads;
      k[u] = i < b1 ? __ldg(keys + i) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k[u] != 0xFFFFFFFFu) atomicAdd(&scnt[(int)(k[u] - lo)], 1);
  }
  __syncthreads();
  // exclusive scan of scnt[0, nr) in place: a contiguous piece per thread + block scan of the sums
  {
    const int per = (nr + kRangeThreads - 1) / kRangeThreads;
    const int j0 = t * per, j1 = j0 + per < nr ? j0 + per : nr;
    int sum = 0;
    for (int j = j0; j < j1; ++j) sum += scnt[j];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int x = s_ws[lane];
      int xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, xi, o);
        if (lane >= o) xi += y;
      }
      s_ws[lane] = xi - x;
    }
    __syncthreads();
    int run = s_ws[warp] + incl - sum;
    for (int j = j0; j < j1; ++j) {
      const int c = scnt[j];
      scnt[j] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int j = t; j < nr; j += kRangeThreads) eoff[lo + j] = b0 + scnt[j];
  if (lo + nr == N && t == 0) eoff[N] = b1;
  __syncthreads();
  for (int64_t i0 = b0 + t; i0 < b1; i0 += (int64_t)U * kRangeThreads) {
    uint32_t k[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * kRangeThreads;
      k[u] = i < b1 ? __ldg(keys + i) : 0xFFFFFFFFu;
      v[u] = i < b1 ? __ldg(vals + i) : 0u;
    }
    int p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) p[u] = k[u] != 0xFFFFFFFFu ? atomicAdd(&scnt[(int)(k[u] - lo)], 1) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (p[u] >= 0) eidx[b0 + p[u]] = (int32_t)v[u];
  }
  __syncthreads();   // scnt[j] = end of node j's segment; the CTA's global writes are visible to it
  if (!SORT) continue;
  for (int j0 = 0; j0 < nr; j0 += kRangeThreads) {
    const int j = j0 + t;
    const bool in = j < nr;
    const int st = in ? (j ? scnt[j - 1] : 0) : 0;
    const int d = in ? scnt[j] - st : 0;
    const bool big = d > kSegMax;
    if (big) giants[atomicAdd(ngiant, 1u)] = (uint32_t)(lo + j);
    const int dd = big ? 0 : d;
    const int wmax = __reduce_max_sync(FULL, (unsigned)dd);
    if (wmax > 1) {
      int32_t* seg = eidx + b0 + st;
      if (wmax <= 8) sort_segment<8>(seg, dd);
      else if (wmax <= 16) sort_segment<16>(seg, dd);
      else if (wmax <= 24) sort_segment<24>(seg, dd);
      else sort_segment<32>(seg, dd);
    }
  }
  }
}

// In-place ascending bitonic sort of each queued segment [off[a], off[a+1]) (shared memory when it
// fits, else directly in global memory), one CTA per segment.
__global__ void __launch_bounds__(1024)
k_segsort_giant(const int64_t* __restrict__ off, int32_t* __restrict__ vals, const uint32_t* __restrict__ giants,
                const unsigned int* __restrict__ ngiant, int smem_cap, const unsigned long long* __restrict__ err) {
  extern __shared__ int32_t sbuf[];
  if (err && *err != ERR_NONE) return;
  const unsigned ng = *ngiant;
  for (unsigned g = blockIdx.x; g < ng; g += gridDim.x) {
    const int64_t a = giants[g];
    const int64_t s = off[a];
    const int64_t n = off[a + 1] - s;
    int32_t* buf = n <= smem_cap ? sbuf : vals + s;
    if (n <= smem_cap)
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sbuf[i] = vals[s + i];
    __syncthreads();
    int64_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int64_t k = 2; k <= n2; k <<= 1) {
      for (int64_t j = k >> 1; j > 0; j >>= 1) {
        for (int64_t t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
          const int64_t blk = t / j, o = t % j;
          int64_t lo, hi;
          if (j == (k >> 1)) { lo = blk * k + o; hi = blk * k + k - 1 - o; }
          else { lo = blk * 2 * j + o; hi = lo + j; }
          if (hi < n) {
            const int32_t x = buf[lo], y = buf[hi];
            if (x > y) { buf[lo] = y; buf[hi] = x; }
          }
        }
        __syncthreads();
      }
    }
    if (n <= smem_cap)
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) vals[s + i] = sbuf[i];
    __syncthreads();
  }
}

// ================================================================================================
// k_elem_offsets: offsets from the stably sorted element-pair keys (no dedupe needed: (node,
// element) pairs are unique once the input is validated).
// ================================================================================================
template <bool ALIGNED>
__global__ void __launch_bounds__(256)
k_elem_offsets(const uint32_t* __restrict__ keys, int64_t n, int64_t N, int64_t* __restrict__ offsets,
               const unsigned long long* __restrict__ err) {
  if (err && *err != ERR_NONE) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 4 * q < n; q += stride) {
    const int64_t i0 = 4 * q;
    uint32_t k[4];
    if (ALIGNED && i0 + 3 < n) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(keys) + q);
      k[0] = x.x; k[1] = x.y; k[2] = x.z; k[3] = x.w;
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) k[r] = (i0 + r < n) ? __ldg(keys + i0 + r) : 0u;
    }
    int64_t prev = i0 == 0 ? -1 : (int64_t)__ldg(keys + i0 - 1);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t i = i0 + r;
      if (i >= n) break;
      const int64_t cur = k[r];
      for (int64_t x = prev + 1; x <= cur; ++x) offsets[x] = i;
      prev = cur;
      if (i == n - 1)
        for (int64_t x = cur + 1; x <= N; ++x) offsets[x] = n;
    }
  }
}

// ================================================================================================
// k_scan_i32: exclusive scan int32 -> int64 (out has n+1 entries), single pass, decoupled
// look-back; warp-striped tiles, warp shuffles inside.
// ================================================================================================
template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
k_scan_i32(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out, uint64_t* status,
           uint32_t* ticket, uint32_t epoch, const unsigned int* __restrict__ guard = nullptr) {
  // Each thread scans ITEMS consecutive counts sequentially (16-byte loads), the warps scan their
  // threads' totals, the block its warps' totals, decoupled look-back across tiles; the exclusive
  // prefixes leave as 16-byte stores (out[i] for i < n), the thread holding item n - 1 writes out[n].
  static_assert(ITEMS % 4 == 0, "vector loads");
  constexpr int WARPS = THREADS / 32;
  if (guard && *guard == 0u) return;   // grid-uniform: a fallback scan that is not needed
  constexpr int TILE = THREADS * ITEMS;
  __shared__ uint64_t s_w[WARPS];
  __shared__ uint64_t s_texcl;
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * TILE + (int64_t)tid * ITEMS;
  int64_t loc[ITEMS];   // inclusive prefix inside the thread
  const bool full = base + ITEMS <= n && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
  if (full) {
    int64_t run = 0;
#pragma unroll
    for (int q = 0; q < ITEMS / 4; ++q) {
      const int4 x = __ldg(reinterpret_cast<const int4*>(in + base) + q);
      run += x.x; loc[4 * q] = run;
      run += x.y; loc[4 * q + 1] = run;
      run += x.z; loc[4 * q + 2] = run;
      run += x.w; loc[4 * q + 3] = run;
    }
  } else {
    int64_t run = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      run += base + k < n ? (int64_t)in[base + k] : 0;
      loc[k] = run;
    }
  }
  const int64_t ttot = loc[ITEMS - 1];
  int64_t winc = ttot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULL, winc, o);
    if (lane >= o) winc += y;
  }
  if (lane == 31) s_w[warp] = (uint64_t)winc;
  __syncthreads();
  if (warp == 0) {
    uint64_t c = lane < WARPS ? s_w[lane] : 0;
    uint64_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const uint64_t tot = __shfl_sync(FULL, incl, 31);
    if (lane < WARPS) s_w[lane] = incl - c;
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed_u64(status, st_pack(epoch, ST_INC, tot));
    } else {
      if (lane == 0) st_relaxed_u64(status + tile, st_pack(epoch, ST_AGG, tot));
      excl = warp_lookback(status, tile, epoch, lane);
      if (lane == 0) st_relaxed_u64(status + tile, st_pack(epoch, ST_INC, excl + tot));
    }
    if (lane == 0) s_texcl = excl;
  }
  __syncthreads();
  const int64_t pre = (int64_t)(s_texcl + s_w[warp]) + winc - ttot;   // sum of every item before base
  if (full && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
    longlong2* o2 = reinterpret_cast<longlong2*>(out + base);
#pragma unroll
    for (int q = 0; q < ITEMS / 2; ++q)
      o2[q] = make_longlong2(pre + (q ? loc[2 * q - 1] : 0), pre + loc[2 * q]);
  } else {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
      if (base + k < n) out[base + k] = pre + (k ? loc[k - 1] : 0);
  }
  if (base < n && base + ITEMS >= n) out[n] = pre + ttot;
}

// ================================================================================================
// Stage kernels for the per-row entry points (emission materialised in slot order).
// ================================================================================================
template <int T, typename KeyT>
__global__ void __launch_bounds__(256)
k_emit_node(const int32_t* __restrict__ conn, int64_t P, int b, KeyT* __restrict__ keys,
            const unsigned long long* __restrict__ err) {
  if (*err != ERR_NONE) return;
  constexpr int K = Elem<T>::K, S = 2 * Elem<T>::E;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / S;
    const int r = (int)(i - e * S);
    int la, lb;
    slot_locals<T>(r, la, lb);
    const uint32_t a = (uint32_t)__ldg(conn + e * K + la);
    const uint32_t v = (uint32_t)__ldg(conn + e * K + lb);
    keys[i] = (KeyT)(((KeyT)a << b) | (KeyT)v);
  }
}

template <int T>
__global__ void __launch_bounds__(256)
k_emit_elem(const int32_t* __restrict__ conn, int64_t P, uint32_t* __restrict__ keys,
            uint32_t* __restrict__ vals, const unsigned long long* __restrict__ err) {
  if (*err != ERR_NONE) return;
  constexpr int K = Elem<T>::K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (uint32_t)__ldg(conn + i);
    vals[i] = (uint32_t)(i / K);
  }
}

// Multi-GPU bucketing: mark, in bucket order, the first incidence of each element inside a bucket
// destined to another rank (flags[j] = 1): those elements' rows travel with the pairs.
__global__ void __launch_bounds__(256)
k_mark_remote_rows(const uint64_t* __restrict__ pairs, int64_t n, uint64_t chunk, int world, int self,
                   int32_t* __restrict__ flags, const unsigned long long* __restrict__ err) {
  if (*err != ERR_NONE) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t p = pairs[j];
    uint64_t g = (p >> 32) / chunk;
    g = g < (uint64_t)world ? g : (uint64_t)world - 1;
    bool f = (int)g != self;
    if (f && j > 0) {
      const uint64_t q = pairs[j - 1];
      uint64_t gq = (q >> 32) / chunk;
      gq = gq < (uint64_t)world ? gq : (uint64_t)world - 1;
      f = !(gq == g && (q & 0xffffffffull) == (p & 0xffffffffull));
    }
    flags[j] = f ? 1 : 0;
  }
}

// Rows per destination: differences of the flag scan at the bucket boundaries (bases[g] = first
// incidence of bucket g).
__global__ void k_row_counts(const int64_t* __restrict__ pos, const uint64_t* __restrict__ bases, int world,
                             int64_t n, unsigned long long* __restrict__ rcnt) {
  const int g = threadIdx.x;
  if (g < world) {
    const int64_t b0 = (int64_t)bases[g], b1 = g + 1 < world ? (int64_t)bases[g + 1] : n;
    rcnt[g] = (unsigned long long)(pos[b1] - pos[b0]);
  }
}

template <int T>
__global__ void __launch_bounds__(256)
k_emit_remote_rows(const uint64_t* __restrict__ pairs, const int32_t* __restrict__ flags,
                   const int64_t* __restrict__ pos, int64_t n, const int32_t* __restrict__ conn, int64_t elem_base,
                   int32_t* __restrict__ relems, int32_t* __restrict__ rrows, const unsigned long long* __restrict__ err) {
  constexpr int K = Elem<T>::K;
  if (*err != ERR_NONE) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[j]) continue;
    const int64_t o = pos[j];
    const int64_t e = (int64_t)(pairs[j] & 0xffffffffull);
    relems[o] = (int32_t)e;
#pragma unroll
    for (int q = 0; q < K; ++q) rrows[o * K + q] = __ldg(conn + (e - elem_base) * K + q);
  }
}

// Chunked mode: add a base to a slice of offsets (local slice offsets -> global CSR offsets).
__global__ void __launch_bounds__(256)
k_shift_offsets(const int64_t* __restrict__ in, int64_t n, int64_t base, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] + base;
}

// Multi-GPU pass 1 for coherent meshes (one read of the shard, grid-stride like k_hist_validate):
// validation (reading R8), the incidence count per owner rank, and the REMOTE incidences (owner !=
// self) appended to rem[] (node << 32 | global element) with one atomic per warp and incidence slot
// — in no particular order; the few remote incidences are put in element order afterwards.
template <int T, int BINS, bool ALIGNED>
__global__ void __launch_bounds__(256)
k_hist_remote(const int32_t* __restrict__ conn, int64_t M, int64_t N, int64_t elem_base, uint64_t owner_div,
              int world, int self, unsigned long long* __restrict__ hist, unsigned long long* __restrict__ err,
              uint64_t* __restrict__ rem, unsigned long long* __restrict__ nrem) {
  constexpr int K = Elem<T>::K;
  __shared__ uint32_t sh[BINS];
  for (int i = threadIdx.x; i < BINS; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int nown = 0;   // own incidences counted in a register (one shared atomic per warp at the end)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < M; base += stride) {
    const int64_t e = base + lane;
    const bool in = e < M;
    int v[K];
    if (in) load_row<T, ALIGNED>(conn, e, v);
    int kind = 0;
    const int bad = in ? row_bad<K>(v, (uint32_t)N, kind) : -1;
    if (in) {
      if (bad >= 0) atomicMin(err, (unsigned long long)err_encode((uint64_t)(elem_base + e), kind, bad));
    }
    const bool ok = in && bad < 0;
    uint32_t rmask = 0;   // incidences of this element owned by another rank
#pragma unroll
    for (int p = 0; p < K; ++p) {
      if (!ok) continue;
      uint64_t o = owner_div <= 0xFFFFFFFFull ? (uint64_t)((uint32_t)v[p] / (uint32_t)owner_div)
                                              : (uint64_t)v[p] / owner_div;
      o = o < (uint64_t)world ? o : (uint64_t)world - 1;
      if ((int)o != self) {
        atomicAdd(&sh[o], 1u);
        rmask |= 1u << p;
      } else {
        ++nown;
      }
    }
    if (__any_sync(FULL, rmask != 0)) {   // rare on a coherent mesh: one atomic per warp and slot
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const bool remote = (rmask >> p) & 1u;
        const unsigned rb = __ballot_sync(FULL, remote);
        if (!rb) continue;
        unsigned long long at = 0;
        if (lane == __ffs(rb) - 1) at = atomicAdd(nrem, (unsigned long long)__popc(rb));
        at = __shfl_sync(FULL, at, __ffs(rb) - 1);
        if (remote)
          rem[at + __popc(rb & lanemask_lt())] = ((uint64_t)(uint32_t)v[p] << 32) | (uint64_t)(elem_base + e);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nown += __shfl_xor_sync(FULL, nown, o);
  if (lane == 0 && nown) atomicAdd(&sh[self], (uint32_t)nown);
  __syncthreads();
  for (int i = threadIdx.x; i < BINS; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// (node << 32 | element) pairs <-> (element - base key, node payload) for sorting the remote
// incidences by element with the u32 onesweep.
__global__ void __launch_bounds__(256)
k_split_pairs(const uint64_t* __restrict__ pairs, int64_t n, int64_t base, uint32_t* __restrict__ keys,
              uint32_t* __restrict__ vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = pairs[i];
    keys[i] = (uint32_t)((int64_t)(q & 0xffffffffull) - base);
    vals[i] = (uint32_t)(q >> 32);
  }
}
__global__ void __launch_bounds__(256)
k_join_pairs(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n, int64_t base,
             uint64_t* __restrict__ pairs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    pairs[i] = ((uint64_t)vals[i] << 32) | (uint64_t)(base + (int64_t)keys[i]);
}

// The incidences an owner finishes, in source-rank order, as up to three pieces: those received
// from lower ranks, its own bucket read in place from the bucketing output (never copied through
// the exchange), those received from higher ranks.  Piece q covers positions [end[q-1], end[q]).
struct PairSrc {
  const uint64_t* p[3];
  int64_t end[3];
  __device__ __forceinline__ uint64_t at(int64_t j) const {
    if (j < end[0]) return p[0][j];
    if (j < end[1]) return p[1][j - end[0]];
    return p[2][j - end[1]];
  }
};
inline PairSrc pair_src(const uint64_t* pairs, int64_t n) { return PairSrc{{pairs, pairs, pairs}, {n, n, n}}; }

// Multi-GPU finish, transpose form (received pairs are element-major, i.e. as coherent as conn):
// distinct nodes per window of 32 consecutive pairs (locality sample), per-node counts, and the
// warp-aggregated scatter of element ids (sorted per node afterwards by k_elem_segsort).
__global__ void __launch_bounds__(256)
k_pairs_locality(PairSrc pairs, int64_t n, unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t j = (int64_t)((double)n * (double)gw / (double)nw) + lane;
  const bool in = j < n;
  const int64_t x = in ? (int64_t)(pairs.at(j) >> 32) : -1;   // one shared sentinel: match cost grows with distinct values
  const unsigned peers = __match_any_sync(FULL, (unsigned long long)x);
  const unsigned g = __reduce_add_sync(FULL, (in && lane == __ffs(peers) - 1) ? 1u : 0u);
  const unsigned act = __popc(__ballot_sync(FULL, in));
  if (lane == 0) {
    atomicAdd(out, (unsigned long long)g);
    atomicAdd(out + 1, (unsigned long long)act);
  }
}



// Chunk-bucketed transpose of received (node << 32 | element) pairs (the multi-GPU finish; the
// scheme of k_chunk_scatter_fixed / k_chunk_sort on the owner's local node ids a - lo).
// FIXED: fixed-capacity buckets [x * cap, (x + 1) * cap), overflow -> *ovf; else (fallback, guarded
// by *ovf) counted buckets at cbase[x] with cursors `cur`.
template <bool FIXED>
__global__ void __launch_bounds__(256)
k_pairs_chunk_scatter(PairSrc pairs, int64_t n, int64_t lo, int cap,
                      const int64_t* __restrict__ cbase, int32_t* __restrict__ cur, int32_t* __restrict__ belem,
                      uint8_t* __restrict__ bnode, unsigned int* __restrict__ ovf) {
  if (!FIXED && *ovf == 0u) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    const int64_t j = base + lane;
    const bool in = j < n;
    const uint64_t p = in ? pairs.at(j) : 0;
    const int a = in ? (int)((int64_t)(p >> 32) - lo) : 0;
    const int x = in ? (a >> kChunkShift) : -1;   // one shared sentinel: match cost grows with distinct values
    const unsigned peers = __match_any_sync(FULL, x);
    const int leader = __ffs(peers) - 1;
    int c = 0;
    if (in && lane == leader) {
      c = atomicAdd(cur + x, (int)__popc(peers));
      if (FIXED && c + (int)__popc(peers) > cap) *ovf = 1u;
    }
    c = __shfl_sync(FULL, c, leader) + __popc(peers & lanemask_lt());
    if (in && (!FIXED || c < cap)) {
      const int64_t pos = (FIXED ? (int64_t)x * cap : cbase[x]) + c;
      belem[pos] = (int32_t)(p & 0xffffffffull);
      bnode[pos] = (uint8_t)(a & (kChunkNodes - 1));
    }
  }
}

// Fallback chunk counts of received pairs (guarded by *ovf).
__global__ void __launch_bounds__(256)
k_pairs_chunk_count(PairSrc pairs, int64_t n, int64_t lo, int32_t* __restrict__ ccnt,
                    const unsigned int* __restrict__ ovf) {
  if (*ovf == 0u) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    const int64_t j = base + lane;
    const bool in = j < n;
    const int x = in ? (int)(((int64_t)(pairs.at(j) >> 32) - lo) >> kChunkShift) : -1;
    const unsigned peers = __match_any_sync(FULL, x);
    if (in && lane == __ffs(peers) - 1) atomicAdd(ccnt + x, (int)__popc(peers));
  }
}

// Multi-GPU finish: local node key and element-id payload of every received pair.
__global__ void __launch_bounds__(256)
k_local_keys(PairSrc pairs, int64_t n, int64_t lo, uint32_t* __restrict__ keys,
             uint32_t* __restrict__ elems) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t p = pairs.at(i);
    keys[i] = (uint32_t)((int64_t)(p >> 32) - lo);
    elems[i] = (uint32_t)(p & 0xffffffffull);
  }
}

}  // namespace mn
