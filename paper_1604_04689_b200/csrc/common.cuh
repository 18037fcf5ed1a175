// common.cuh — shared device definitions of libmeshnbr (sm_100a only).
//
// Nothing here is shared with oracle/: the element tables below are this side's own encoding of
// DESIGN.md reading R4/R5 (edge lists) — see the comments next to each literal.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "meshnbr.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libmeshnbr is written for sm_100a (B200) only"
#endif

namespace mn {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t ERR_NONE = ~0ull;

// ------------------------------------------------------------------------------------------------
// Validation word: the lowest (element, kind, position) wins an atomicMin.
//   word = elem << 5 | kind << 4 | pos ; kind 0 = index out of range, 1 = repeated node (R8)
// ------------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t err_encode(uint64_t elem, int kind, int pos) {
  return (elem << 5) | ((uint64_t)kind << 4) | (uint64_t)pos;
}

// ------------------------------------------------------------------------------------------------
// Look-back status words (decoupled look-back, Merrill & Garland 2016 / onesweep, Adinets &
// Merrill 2022).  64-bit so a digit bucket may exceed 2^30 pairs (config 5 has 2.36e9 pairs):
//   [63:56] epoch (pass number + 1; a word from an earlier pass reads as "not ready")
//   [55:54] flag  (1 = tile aggregate, 2 = inclusive prefix)
//   [53:0]  value
// ------------------------------------------------------------------------------------------------
constexpr uint64_t ST_AGG = 1, ST_INC = 2;
constexpr uint64_t ST_VMASK = (1ull << 54) - 1;

__device__ __forceinline__ uint64_t st_pack(uint32_t epoch, uint64_t flag, uint64_t v) {
  return ((uint64_t)epoch << 56) | (flag << 54) | v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Wait for the status word of one predecessor and return (flag, value).
__device__ __forceinline__ uint64_t lookback_wait(const uint64_t* p, uint32_t epoch) {
  uint64_t w = ld_relaxed_u64(p);
  int spins = 0;
  while ((uint32_t)(w >> 56) != epoch || ((w >> 54) & 3u) == 0) {
    if (++spins > 4) __nanosleep(32);
    w = ld_relaxed_u64(p);
  }
  return w;
}

// Windowed decoupled look-back for BPT digits owned by this thread: W predecessor status words per
// digit are requested at once, so a walk over k aggregate-only tiles costs ceil(k / W) round trips
// to L2 instead of k.  status is [tiles][bins]; returns the exclusive prefix of each digit.
template <int BPT, int W>
__device__ __forceinline__ void lookback_issue(const uint64_t* status, int bins, uint32_t tile, int b0,
                                               uint64_t (&w)[BPT][W]) {
  const int64_t t0 = (int64_t)tile - 1;
#pragma unroll
  for (int j = 0; j < BPT; ++j)
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int64_t t = t0 - k;
      w[j][k] = t >= 0 ? ld_relaxed_u64(status + (size_t)t * bins + b0 + j) : 0;
    }
}

template <int BPT, int W>
__device__ __forceinline__ void lookback_finish(const uint64_t* status, int bins, uint32_t tile, int b0,
                                                uint32_t epoch, uint64_t (&w)[BPT][W], uint64_t (&excl)[BPT]) {
  const int64_t t0 = (int64_t)tile - 1;
#pragma unroll
  for (int j = 0; j < BPT; ++j) {
    excl[j] = 0;
    int64_t tb = t0;
    bool done = false;
    while (true) {
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (!done) {
          const uint64_t* p = status + (size_t)(tb - k) * bins + b0 + j;
          uint64_t x = w[j][k];
          int spins = 0;
          while ((uint32_t)(x >> 56) != epoch || ((x >> 54) & 3u) == 0) {
            if (++spins > 2) __nanosleep(16);
            x = ld_relaxed_u64(p);
          }
          excl[j] += x & ST_VMASK;
          done = ((x >> 54) & 3u) == ST_INC;
        }
      }
      if (done) break;
      tb -= W;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int64_t t = tb - k;
        w[j][k] = t >= 0 ? ld_relaxed_u64(status + (size_t)t * bins + b0 + j) : 0;
      }
    }
  }
}

// Windowed decoupled look-back for BPT digits owned by this thread: W predecessor status words per
// digit are requested at once, so a walk over k aggregate-only tiles costs ceil(k / W) round trips
// to L2 instead of k.  status is [tiles][bins]; returns the exclusive prefix of each digit.
template <int BPT, int W>
__device__ __forceinline__ void lookback_bins(const uint64_t* status, int bins, uint32_t tile, int b0,
                                              uint32_t epoch, uint64_t (&excl)[BPT]) {
  uint64_t w[BPT][W];
  lookback_issue<BPT, W>(status, bins, tile, b0, w);
  lookback_finish<BPT, W>(status, bins, tile, b0, epoch, w, excl);
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp-cooperative look-back over one status word per tile (compaction / scan kernels): the 32
// lanes read 32 predecessors per round trip.  Call with the whole warp; returns the exclusive
// prefix in every lane.
__device__ __forceinline__ uint64_t warp_lookback(const uint64_t* status, uint32_t tile, uint32_t epoch,
                                                  int lane) {
  uint64_t excl = 0;
  int64_t tb = (int64_t)tile - 1;
  while (true) {
    const int64_t t = tb - lane;
    uint64_t x = t >= 0 ? ld_relaxed_u64(status + t) : st_pack(epoch, ST_INC, 0);
    while (true) {
      const bool ready = (uint32_t)(x >> 56) == epoch && ((x >> 54) & 3u) != 0;
      if (__all_sync(0xffffffffu, ready)) break;
      if (!ready) {
        __nanosleep(16);
        x = ld_relaxed_u64(status + t);
      }
    }
    const unsigned inc = __ballot_sync(0xffffffffu, ((x >> 54) & 3u) == ST_INC);
    uint64_t v = x & ST_VMASK;
    if (inc) {
      const int first = __ffs(inc) - 1;   // nearest predecessor holding an inclusive prefix
      if (lane > first) v = 0;
      return excl + warp_sum_u64(v);
    }
    excl += warp_sum_u64(v);
    tb -= 32;
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- bulk asynchronous copies (TMA 1-D, cp.async.bulk) into shared memory, mbarrier completion ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");   // visible to the async proxy
}
// arrive (one of the init count) and expect `bytes` of transactions on the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// global -> shared bulk copy: dst, src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n MN_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MN_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Streaming loads that do not pollute L1 (each key is read exactly once per pass).
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// 16-byte read-only load with the L2 fill limited to 64 bytes (random row gathers: the default fill
// brings more sectors than the one row needs)
__device__ __forceinline__ int4 ldg_l2_64(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L2::64B.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// ------------------------------------------------------------------------------------------------
// Element types.  For node pairs, slot r in [0, 2E) of an element holds (conn[la(r)], conn[lb(r)]):
// r = 2j is edge j forward, r = 2j+1 edge j reversed (R5).  la/lb are 4-bit local
// indices packed into 128-bit literals (slot r at bits 4r..4r+3).
// ------------------------------------------------------------------------------------------------
template <int T> struct Elem;
template <> struct Elem<MN_TRI3> {   // edges (0,1) (1,2) (2,0)
  static constexpr int K = 3, E = 3, C = 2;          // C = edges incident to each local node
  static constexpr uint64_t A_LO = 0x22110ull, A_HI = 0, B_LO = 0x201201ull, B_HI = 0;
};
template <> struct Elem<MN_QUAD4> {  // ring edges (0,1) (1,2) (2,3) (3,0), no diagonals
  static constexpr int K = 4, E = 4, C = 2;
  static constexpr uint64_t A_LO = 0x3322110ull, A_HI = 0, B_LO = 0x30231201ull, B_HI = 0;
};
template <> struct Elem<MN_TET4> {   // (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
  static constexpr int K = 4, E = 6, C = 3;
  static constexpr uint64_t A_LO = 0x323121302010ull, A_HI = 0, B_LO = 0x231312030201ull, B_HI = 0;
};
template <> struct Elem<MN_HEX8> {   // VTK: (0,1)(1,2)(2,3)(3,0)(4,5)(5,6)(6,7)(7,4)(0,4)(1,5)(2,6)(3,7)
  static constexpr int K = 8, E = 12, C = 3;
  static constexpr uint64_t A_LO = 0x4776655403322110ull, A_HI = 0x73625140ull,
                            B_LO = 0x7467564530231201ull, B_HI = 0x37261504ull;
};

// Validation of one element row (R8): the lowest offending position, an index outside
// [0, N) before a repeated node (kind 0 / 1), or -1.  N <= INT32_MAX (checked at the C ABI), so one
// unsigned compare per entry covers both bounds; the common valid row costs one OR-chain of
// compares and the position is only worked out for a bad row.
template <int K>
__device__ __forceinline__ int row_bad(const int (&v)[K], uint32_t N, int& kind) {
  bool any = false;
#pragma unroll
  for (int p = 0; p < K; ++p) any |= (uint32_t)v[p] >= N;
#pragma unroll
  for (int p = 1; p < K; ++p)
#pragma unroll
    for (int q = 0; q < p; ++q) any |= v[q] == v[p];
  kind = 0;
  if (!any) return -1;
  int bad = -1;
#pragma unroll
  for (int p = K - 1; p >= 0; --p)
    if ((uint32_t)v[p] >= N) bad = p;
  if (bad >= 0) return bad;
#pragma unroll
  for (int p = K - 1; p >= 1; --p) {
    bool dup = false;
#pragma unroll
    for (int q = 0; q < p; ++q) dup |= (v[q] == v[p]);
    if (dup) bad = p;
  }
  kind = 1;
  return bad;
}

template <int T>
__device__ __forceinline__ void slot_locals(int r, int& la, int& lb) {
  using EL = Elem<T>;
  if (EL::A_HI == 0 || r < 16) {
    la = (int)((EL::A_LO >> (4 * r)) & 0xF);
    lb = (int)((EL::B_LO >> (4 * r)) & 0xF);
  } else {
    la = (int)((EL::A_HI >> (4 * (r - 16))) & 0xF);
    lb = (int)((EL::B_HI >> (4 * (r - 16))) & 0xF);
  }
}

// Edge-neighbours of each local node (derived from the same edge lists): local node p's C
// neighbours are nibbles p*C .. p*C+C-1 of (NB_LO | NB_HI << 64).
template <int T> struct Nbr;
template <> struct Nbr<MN_TRI3> { static constexpr uint64_t LO = 0x102021ull, HI = 0; };           // {1,2} {0,2} {0,1}
template <> struct Nbr<MN_QUAD4> { static constexpr uint64_t LO = 0x20312031ull, HI = 0; };        // {1,3} {0,2} {1,3} {0,2}
template <> struct Nbr<MN_TET4> { static constexpr uint64_t LO = 0x210310320321ull, HI = 0; };     // all other three
template <> struct Nbr<MN_HEX8> {   // {1,3,4} {0,2,5} {1,3,6} {0,2,7} {0,5,7} {1,4,6} {2,5,7} {3,4,6}
  static constexpr uint64_t LO = 0x1750720631520431ull, HI = 0x64375264ull;
};

template <int T>
__device__ __forceinline__ int nbr_local(int p, int c) {
  const int i = p * Elem<T>::C + c;
  if constexpr (Nbr<T>::HI == 0) {
    return (int)((Nbr<T>::LO >> (4 * i)) & 0xF);
  } else {
    return (int)(((i < 16) ? (Nbr<T>::LO >> (4 * i)) : (Nbr<T>::HI >> (4 * (i - 16)))) & 0xF);
  }
}

inline int arity_of(int t) { return t == MN_TRI3 ? 3 : (t == MN_HEX8 ? 8 : 4); }
inline int edges_of(int t) { return t == MN_TRI3 ? 3 : t == MN_QUAD4 ? 4 : t == MN_TET4 ? 6 : 12; }

// Bits of a node id: b = max(1, bit_length(N - 1)) (R11).
inline int node_bits(int64_t N) {
  int b = 0;
  uint64_t x = N > 1 ? (uint64_t)(N - 1) : 0;
  while (x) { ++b; x >>= 1; }
  return b < 1 ? 1 : b;
}

}  // namespace mn
