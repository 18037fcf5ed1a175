// poly.cuh — polygon / mixed-arity surface meshes (the paper's title
// "generic meshes", §2.2 "applicable to arbitrary meshes"; SPEC.md Mesh
// element_kind Polygon).
//
// A polygon mesh is a CSR connectivity: element e is the ring idx[off[e]], ..., idx[off[e+1]-1]
// with arity k_e = off[e+1] - off[e] >= 3; its edges are consecutive ring entries plus the closing
// edge (SPEC Element: "order defines the edge ring").  The same pipeline as the fixed types'
// transpose path, with variable-length rows:
//   k_poly_count    validation (reading R18) + per-node incidence counts (+ raw candidate counts
//                   for the element-sharing adjacency: k_e - 1 per incidence)
//   k_scan_i32      offsets of the element CSR (and of the raw candidate regions)
//   k_poly_scatter  element ids into the element CSR (warp-aggregated atomics), then
//   k_elem_segsort  the shared per-node segment sort restores ascending element ids
//   k_poly_gather   per node: the candidates of each incident ring (the two ring neighbours, or all
//                   other ring nodes) into a private shared-memory hash set, sorted, packed per
//                   128-node chunk; nodes with more than kMaxUnique distinct neighbours go to
//   k_poly_giant    one CTA per node: bitonic sort + dedupe of its raw candidates
//   k_node_compact  (shared with the fixed types) packs the node lists into the output CSR
#pragma once

#include "kernels.cuh"

namespace mn {

// Polygon validation word: elem << 24 | kind << 22 | pos (22 bits).  Kinds: 0 index out of range,
// 1 repeated node, 2 arity < 3, 3 malformed offsets / arity beyond kPolyMaxArity.
constexpr int64_t kPolyMaxArity = (1 << 22) - 1;
__host__ __device__ __forceinline__ uint64_t poly_err(uint64_t elem, int kind, int64_t pos) {
  return (elem << 24) | ((uint64_t)kind << 22) | (uint64_t)(pos & 0x3FFFFF);
}

// One thread per element (grid-stride).  Per element, in order (R18): offsets inside
// [0, conn_len] and arity <= kPolyMaxArity, arity >= 3, every index in [0, N), no repeated index
// (first repeated position).  Valid elements add 1 per node to cnt and, when raw != nullptr,
// k_e - 1 per node to raw (element-sharing candidates).
__global__ void __launch_bounds__(256)
k_poly_count(const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t M, int64_t conn_len,
             int64_t N, int32_t* __restrict__ cnt, int32_t* __restrict__ raw, unsigned long long* __restrict__ err) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < M; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[e], k = off[e + 1] - b;
    if (b < 0 || off[e + 1] > conn_len || k > kPolyMaxArity) {
      atomicMin(err, (unsigned long long)poly_err(e, 3, 0));
      continue;
    }
    if (k < 3) {
      atomicMin(err, (unsigned long long)poly_err(e, 2, 0));
      continue;
    }
    const int32_t* row = idx + b;
    int64_t bad = -1;
    for (int64_t p = 0; p < k && bad < 0; ++p)
      if (row[p] < 0 || (int64_t)row[p] >= N) bad = p;
    if (bad >= 0) {
      atomicMin(err, (unsigned long long)poly_err(e, 0, bad));
      continue;
    }
    for (int64_t p = 1; p < k && bad < 0; ++p) {
      const int32_t x = row[p];
      for (int64_t q = 0; q < p; ++q)
        if (row[q] == x) { bad = p; break; }
    }
    if (bad >= 0) {
      atomicMin(err, (unsigned long long)poly_err(e, 1, bad));
      continue;
    }
    for (int64_t p = 0; p < k; ++p) {
      atomicAdd(cnt + row[p], 1);
      if (raw) atomicAdd(raw + row[p], (int)(k - 1));
    }
  }
}

// Lane per element, the warp steps through local positions together; lanes holding the same node
// at the same step reserve their slots with one returning atomic (consecutive elements of a mesh
// numbered with locality share nodes).  Order inside a node's list is fixed by k_elem_segsort.
__global__ void __launch_bounds__(256)
k_poly_scatter(const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t M,
               const int64_t* __restrict__ eoff, int32_t* __restrict__ cursor, int32_t* __restrict__ eidx,
               const unsigned long long* __restrict__ err) {
  if (*err != ERR_NONE) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < M; base += stride) {
    const int64_t e = base + lane;
    const bool in = e < M;
    const int64_t b = in ? off[e] : 0;
    const int k = in ? (int)(off[e + 1] - b) : 0;
    const int kmax = (int)__reduce_max_sync(FULL, (unsigned)k);
    for (int p = 0; p < kmax; ++p) {
      const bool mine = p < k;
      const int x = mine ? idx[b + p] : -1;   // one shared sentinel: match cost grows with distinct values
      const unsigned peers = __match_any_sync(FULL, x);
      const int leader = __ffs(peers) - 1;
      int c = 0;
      if (mine && lane == leader) c = atomicAdd(cursor + x, (int)__popc(peers));
      c = __shfl_sync(FULL, c, leader);
      if (mine) eidx[eoff[x] + c + __popc(peers & lanemask_lt())] = (int32_t)e;
    }
  }
}

// ---- chunk-bucketed polygon transpose (node / element outputs; the fixed types' scheme, kernels.cuh)
// Validation of one ring (reading R18, the order of k_poly_count): returns -1 if valid, else the
// error word's (kind, pos) packed as kind << 22 | pos.
__device__ __forceinline__ int64_t poly_check(const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                                              int64_t e, int64_t L, int64_t N) {
  const int64_t b = off[e], k = off[e + 1] - b;
  if (b < 0 || off[e + 1] > L || k > kPolyMaxArity) return (int64_t)3 << 22;
  if (k < 3) return (int64_t)2 << 22;
  const int32_t* row = idx + b;
  for (int64_t p = 0; p < k; ++p)
    if (row[p] < 0 || (int64_t)row[p] >= N) return p;
  for (int64_t p = 1; p < k; ++p) {
    const int32_t x = row[p];
    for (int64_t q = 0; q < p; ++q)
      if (row[q] == x) return ((int64_t)1 << 22) | p;
  }
  return -1;
}

// FIXED: single read, validation + append (element id, local node byte) to the node's 128-node
// chunk bucket at [x * cap, (x + 1) * cap); an overflow sets *ovf (the guarded counted path then
// replaces the result).  !FIXED (fallback, guarded by *ovf): counted buckets at cbase[x], cursors
// `cur`.  Lane per element; the warp steps through ring positions together and lanes holding the
// same chunk at a step reserve their slots with one returning atomic.
template <bool FIXED>
__global__ void __launch_bounds__(256)
k_poly_chunk_scatter(const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t M, int64_t L,
                     int64_t N, int cap, const int64_t* __restrict__ cbase, int32_t* __restrict__ cur,
                     int32_t* __restrict__ belem, uint8_t* __restrict__ bnode, unsigned long long* __restrict__ err,
                     unsigned int* __restrict__ ovf) {
  if (!FIXED && *ovf == 0u) return;
  if (!FIXED && *err != ERR_NONE) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < M; base += stride) {
    const int64_t e = base + lane;
    bool ok = e < M;
    if (FIXED && ok) {
      const int64_t c = poly_check(off, idx, e, L, N);
      if (c >= 0) {
        atomicMin(err, (unsigned long long)poly_err((uint64_t)e, (int)(c >> 22), c & 0x3FFFFF));
        ok = false;
      }
    }
    const int64_t b = ok ? off[e] : 0;
    const int k = ok ? (int)(off[e + 1] - b) : 0;
    const int kmax = (int)__reduce_max_sync(FULL, (unsigned)k);
    for (int p = 0; p < kmax; ++p) {
      const bool mine = p < k;
      const int v = mine ? idx[b + p] : 0;
      const int x = mine ? (v >> kChunkShift) : -1;   // one shared sentinel: match cost grows with distinct values
      const unsigned peers = __match_any_sync(FULL, x);
      const int leader = __ffs(peers) - 1;
      int c = 0;
      if (mine && lane == leader) {
        c = atomicAdd(cur + x, (int)__popc(peers));
        if (FIXED && c + (int)__popc(peers) > cap) *ovf = 1u;
      }
      c = __shfl_sync(FULL, c, leader) + __popc(peers & lanemask_lt());
      if (mine && (!FIXED || c < cap)) {
        const int64_t pos = (FIXED ? (int64_t)x * cap : cbase[x]) + c;
        belem[pos] = (int32_t)e;
        bnode[pos] = (uint8_t)(v & (kChunkNodes - 1));
      }
    }
  }
}

// Fallback counts (guarded by *ovf): per-chunk incidence counts of the (already validated) rings.
__global__ void __launch_bounds__(256)
k_poly_chunk_count(const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t M,
                   int32_t* __restrict__ ccnt, const unsigned long long* __restrict__ err,
                   const unsigned int* __restrict__ ovf) {
  if (*ovf == 0u || *err != ERR_NONE) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < M; base += stride) {
    const int64_t e = base + lane;
    const bool in = e < M;
    const int64_t b = in ? off[e] : 0;
    const int k = in ? (int)(off[e + 1] - b) : 0;
    const int kmax = (int)__reduce_max_sync(FULL, (unsigned)k);
    for (int p = 0; p < kmax; ++p) {
      const bool mine = p < k;
      const int x = mine ? (idx[b + p] >> kChunkShift) : -1;
      const unsigned peers = __match_any_sync(FULL, x);
      if (mine && lane == __ffs(peers) - 1) atomicAdd(ccnt + x, (int)__popc(peers));
    }
  }
}

// Raw candidate region of node a: rawoff ? [rawoff[a], rawoff[a+1]) : C * [eoff[a], eoff[a+1]).
__device__ __forceinline__ int64_t poly_raw_base(const int64_t* eoff, const int64_t* rawoff, int C, int64_t a) {
  return rawoff ? rawoff[a] : (int64_t)C * eoff[a];
}

// Candidates of node a from ring (row, k): SHARED: all other ring nodes; else the two ring
// neighbours of a's position.  f(v) is called per candidate.
template <bool SHARED, typename F>
__device__ __forceinline__ void poly_candidates(const int32_t* __restrict__ row, int k, int32_t a, F&& f) {
  if (SHARED) {
    for (int q = 0; q < k; ++q) {
      const int32_t v = __ldg(row + q);
      if (v != a) f((uint32_t)v);
    }
  } else {
    int p = 0;
    while (__ldg(row + p) != a) ++p;   // a is in the ring: it was found through the element CSR
    f((uint32_t)__ldg(row + (p == 0 ? k - 1 : p - 1)));
    f((uint32_t)__ldg(row + (p == k - 1 ? 0 : p + 1)));
  }
}

// Per-node hash-set expansion, the polygon counterpart of k_node_gather_t (same shared-memory
// set, dense per-chunk layout and giant hand-off; see kernels.cuh).
template <bool SHARED>
__global__ void __launch_bounds__(kNodeThreads)
k_poly_gather(const int64_t* __restrict__ eoff, const int32_t* __restrict__ eidx, const int64_t* __restrict__ off,
              const int32_t* __restrict__ idx, int64_t N, const int64_t* __restrict__ rawoff, int C,
              uint32_t* __restrict__ temp, int32_t* __restrict__ cnt, int32_t* __restrict__ lofs,
              uint32_t* __restrict__ giants, unsigned int* __restrict__ ngiant,
              const unsigned long long* __restrict__ err) {
  constexpr uint32_t EMPTY = 0xFFFFFFFFu;
  constexpr int HB = 5, HS = 1 << HB, MU = kMaxUnique;
  __shared__ uint32_t tab[HS][kNodeThreads];
  __shared__ uint32_t s_wsum[kNodeThreads / 32];
  if (err && *err != ERR_NONE) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * kNodeThreads;
  const int64_t a = n0 + t;
  const bool valid = a < N;
  int L = 0;
  uint32_t used = 0;
  int64_t raw = 0;
  if (valid) {
    raw = poly_raw_base(eoff, rawoff, C, a + 1) - poly_raw_base(eoff, rawoff, C, a);
#pragma unroll
    for (int i = 0; i < HS; ++i) tab[i][t] = EMPTY;
    const int64_t s0 = eoff[a], s1 = eoff[a + 1];
    auto insert = [&](uint32_t v) {
      uint32_t h = (v * 0x9E3779B1u) >> (32 - HB);
      while (L <= MU) {
        const uint32_t x = tab[h][t];
        if (x == v) break;
        if (x == EMPTY) {
          tab[h][t] = v;
          used |= 1u << h;
          ++L;
          break;
        }
        h = (h + 1) & (HS - 1);
      }
    };
    if (SHARED) {
      for (int64_t i = s0; i < s1 && L <= MU; ++i) {
        const int32_t e = eidx[i];
        const int64_t b = off[e];
        poly_candidates<SHARED>(idx + b, (int)(off[e + 1] - b), (int32_t)a, insert);
      }
    } else {
      // ring-edge candidates, B incidences in flight: element ids, ring bounds and the first four
      // ring entries are independent loads; rings of arity <= 4 are resolved in registers
      constexpr int B = 4;
      for (int64_t i0 = s0; i0 < s1 && L <= MU; i0 += B) {
        int32_t e[B];
#pragma unroll
        for (int q = 0; q < B; ++q) e[q] = i0 + q < s1 ? __ldg(eidx + i0 + q) : -1;
        int64_t rb[B];
        int rk[B];
#pragma unroll
        for (int q = 0; q < B; ++q) {
          rb[q] = e[q] >= 0 ? __ldg(off + e[q]) : 0;
          rk[q] = e[q] >= 0 ? (int)(__ldg(off + e[q] + 1) - rb[q]) : 0;
        }
        int32_t r[B][4];
#pragma unroll
        for (int q = 0; q < B; ++q)
#pragma unroll
          for (int j = 0; j < 4; ++j) r[q][j] = j < rk[q] ? __ldg(idx + rb[q] + j) : -1;
#pragma unroll
        for (int q = 0; q < B; ++q) {
          if (e[q] < 0) continue;
          const int k = rk[q];
          if (k <= 4) {
            const int32_t* x = r[q];
            const int p = x[0] == (int32_t)a ? 0 : x[1] == (int32_t)a ? 1 : x[2] == (int32_t)a ? 2 : 3;
            const int pp = p == 0 ? k - 1 : p - 1, pn = p == k - 1 ? 0 : p + 1;
            insert((uint32_t)(pp == 0 ? x[0] : pp == 1 ? x[1] : pp == 2 ? x[2] : x[3]));
            insert((uint32_t)(pn == 0 ? x[0] : pn == 1 ? x[1] : pn == 2 ? x[2] : x[3]));
          } else {
            poly_candidates<false>(idx + rb[q], k, (int32_t)a, insert);
          }
        }
      }
    }
  }
  const bool giant = valid && L > MU;
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
  const int lmax = (int)__reduce_max_sync(FULL, giant ? 0u : (unsigned)L);
  if (!valid) return;
  lofs[a] = (int32_t)excl;
  if (giant) {
    giants[atomicAdd(ngiant, 1u)] = (uint32_t)a;
    return;
  }
  int w = 0;
  while (used) {
    const int i = __ffs((int)used) - 1;
    used &= used - 1;
    tab[w++][t] = tab[i][t];
  }
  uint32_t* out = temp + poly_raw_base(eoff, rawoff, C, n0) + excl;
  if (lmax <= 8) sort_small<8, HS>(tab, t, L, out);
  else if (lmax <= 16) sort_small<16, HS>(tab, t, L, out);
  else sort_small<32, HS>(tab, t, L, out);
  cnt[a] = L;
}

// One CTA per giant node: its raw candidates (smem when they fit, else its reserved global raw
// slots), block bitonic sort, dedupe into the reserved slot.
template <bool SHARED>
__global__ void __launch_bounds__(1024)
k_poly_giant(const int64_t* __restrict__ eoff, const int32_t* __restrict__ eidx, const int64_t* __restrict__ off,
             const int32_t* __restrict__ idx, const int64_t* __restrict__ rawoff, int C, uint32_t* __restrict__ temp,
             int32_t* __restrict__ cnt, const int32_t* __restrict__ lofs, const uint32_t* __restrict__ giants,
             const unsigned int* __restrict__ ngiant, int smem_cap, const unsigned long long* __restrict__ err) {
  extern __shared__ uint32_t sv[];
  __shared__ unsigned long long s_fill;
  if (err && *err != ERR_NONE) return;
  const unsigned ng = *ngiant;
  for (unsigned g = blockIdx.x; g < ng; g += gridDim.x) {
    const int64_t a = giants[g];
    const int64_t s = eoff[a], d = eoff[a + 1] - s;
    const int64_t raw = poly_raw_base(eoff, rawoff, C, a + 1) - poly_raw_base(eoff, rawoff, C, a);
    const int64_t n0 = (a / kNodeThreads) * kNodeThreads;
    uint32_t* out = temp + poly_raw_base(eoff, rawoff, C, n0) + lofs[a];
    uint32_t* buf = raw <= smem_cap ? sv : out;
    if (threadIdx.x == 0) s_fill = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
      const int32_t e = eidx[s + i];
      const int64_t b = off[e];
      const int k = (int)(off[e + 1] - b);
      const int64_t at = (int64_t)atomicAdd(&s_fill, (unsigned long long)(SHARED ? k - 1 : 2));
      int c = 0;
      poly_candidates<SHARED>(idx + b, k, (int32_t)a, [&](uint32_t v) { buf[at + (c++)] = v; });
    }
    __syncthreads();
    const int u = block_sort_dedupe(buf, raw, out);
    if (threadIdx.x == 0) cnt[a] = u;
    __syncthreads();
  }
}

}  // namespace mn
