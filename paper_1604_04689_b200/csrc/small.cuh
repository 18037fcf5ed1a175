// small.cuh — the latency path for small meshes (configs 1-like: a few thousand elements), included
// by meshnbr.cu after kernels.cuh.  The staged pipeline costs ~10 launches, several memsets and
// allocations for a mesh that fits in one SM's shared memory; here ONE CTA runs every row of
// SURVEY §8(a) for both outputs:
//   a1/a2 validation (lowest element wins, reading R8) + per-node incidence counts   (smem atomics)
//   a5    exclusive scan -> element-CSR offsets                                       (block scan)
//   a3e   scatter of the element ids into their node segments + per-segment sort      (smem)
//   a3n/a4 per node: its C * deg candidate neighbours (the rows of its elements), sorted and
//         deduplicated in place (the paper's sort + adjacent difference, per segment)
//   a5    exclusive scan of the distinct counts -> node-CSR offsets, lists packed
// The node lists are packed straight into the node-index output (capacity C * Pe) and the kernel
// writes (error word, node nnz, fallback flag) into pinned host memory: one launch, one sync.  A node with more than kSmallMaxCand candidates (or an element list
// longer than kSmallMaxDeg) sets the fallback flag and the call reruns on the staged path.
#pragma once

namespace mn {

constexpr int kSmallThreads = 1024;
constexpr int64_t kSmallMaxN = 4096;          // nodes (3 int arrays of N + 1 in shared memory)
constexpr int64_t kSmallMaxPe = 8192;         // incidences (element lists + C * Pe candidates in smem)
constexpr int kSmallMaxCand = 160;            // per-node candidates sorted by one thread
constexpr int kSmallMaxDeg = 160;             // per-node element-list length sorted by one thread

inline size_t small_smem_bytes(int64_t N, int64_t Pe, int C) {
  return (size_t)(3 * (N + 1) + 2 * Pe + (int64_t)C * Pe + 64) * 4;
}

// In-place exclusive scan of a[0, n) (n <= 8 * blockDim), total to a[n]; all threads call it.
__device__ __forceinline__ void small_block_scan(int* a, int n, int* wsum) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int j0 = min(n, t * per), j1 = min(n, j0 + per);
  int sum = 0;
  for (int j = j0; j < j1; ++j) sum += a[j];
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int x = lane < nw ? wsum[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < nw) wsum[lane] = xi - x;
    if (lane == 31) wsum[32] = xi;
  }
  __syncthreads();
  int run = wsum[warp] + incl - sum;
  for (int j = j0; j < j1; ++j) {
    const int c = a[j];
    a[j] = run;
    run += c;
  }
  if (t == 0) a[n] = wsum[32];
  __syncthreads();
}

template <typename V>
__device__ __forceinline__ void small_isort(V* v, int n) {
  for (int i = 1; i < n; ++i) {
    const V x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
}

// Sort + adjacent-difference dedupe of seg[0, m) (m <= NET) in registers; distinct values back to
// seg[0, L).  Returns L.
template <int NET>
__device__ __forceinline__ int small_sort_unique(uint32_t* seg, int m) {
  int32_t v[NET];
#pragma unroll
  for (int i = 0; i < NET; ++i) v[i] = i < m ? (int32_t)seg[i] : INT32_MAX;
  oddeven_sort<NET>(v);
  int L = 0;
#pragma unroll
  for (int i = 0; i < NET; ++i)
    if (i < m && (i == 0 || v[i] != v[i - 1])) seg[L++] = (uint32_t)v[i];
  return L;
}

// ctrl (pinned host memory, written directly): [0] error word (ERR_NONE if valid), [1] node nnz,
// [2] fallback flag.  fin: the node CSR indices (capacity C * Pe, packed in node order).
template <int T, bool ALIGNED>
__global__ void __launch_bounds__(kSmallThreads, 1)
k_small_both(const int32_t* __restrict__ conn, int M, int N, int64_t* __restrict__ elem_off,
             int32_t* __restrict__ elem_idx, int64_t* __restrict__ node_off, uint32_t* __restrict__ fin,
             unsigned long long* __restrict__ ctrl) {
  constexpr int K = Elem<T>::K, C = Elem<T>::C;
  constexpr bool simplex = (C == K - 1);
  extern __shared__ int sm[];
  int* s_off = sm;                 // N + 1: counts -> element-CSR offsets
  int* s_cur = s_off + N + 1;      // N + 1: scatter cursors
  int* s_ncnt = s_cur + N + 1;     // N + 1: node distinct counts -> node-CSR offsets
  int* s_el = s_ncnt + N + 1;      // Pe: element ids by node
  int* s_conn = s_el + M * K;      // Pe: the connectivity, read from global memory once
  uint32_t* raw = reinterpret_cast<uint32_t*>(s_conn + M * K);   // C * Pe: candidate segments at C * eoff[v]
  __shared__ int s_ws[33];
  __shared__ unsigned long long s_err;
  __shared__ int s_big;
  const int t = threadIdx.x;
  for (int v = t; v <= N; v += blockDim.x) s_off[v] = 0;
  if (t == 0) { s_err = ERR_NONE; s_big = 0; }
  __syncthreads();
  // ---- a1/a2: validation (R8) + incidence counts ----
  for (int e = t; e < M; e += blockDim.x) {
    int row[K];
    load_row<T, ALIGNED>(conn, e, row);
#pragma unroll
    for (int p = 0; p < K; ++p) s_conn[e * K + p] = row[p];
    int kind = 0;
    const int bad = row_bad<K>(row, (uint32_t)N, kind);
    if (bad >= 0) {
      atomicMin(&s_err, (unsigned long long)err_encode((uint64_t)e, kind, bad));
    } else {
#pragma unroll
      for (int p = 0; p < K; ++p) atomicAdd(&s_off[row[p]], 1);
    }
  }
  __syncthreads();
  if (s_err != ERR_NONE) {
    if (t == 0) { ctrl[0] = s_err; ctrl[1] = 0; ctrl[2] = 0; }
    return;
  }
  // ---- a5 (elements): offsets ----
  small_block_scan(s_off, N, s_ws);
  for (int v = t; v <= N; v += blockDim.x) {
    s_cur[v] = s_off[v];
    if (elem_off) elem_off[v] = s_off[v];
  }
  __syncthreads();
  // ---- a3e: element ids into their node segments, each segment sorted ----
  for (int i = t; i < M * K; i += blockDim.x) s_el[atomicAdd(&s_cur[s_conn[i]], 1)] = i / K;
  __syncthreads();
  for (int v = t; v < N; v += blockDim.x) {
    const int b = s_off[v], d = s_off[v + 1] - b;
    if (d > kSmallMaxDeg) { s_big = 1; continue; }
    if (d <= 8) sort_segment<8>(s_el + b, d);
    else if (d <= 16) sort_segment<16>(s_el + b, d);
    else if (d <= 32) sort_segment<32>(s_el + b, d);
    else small_isort(s_el + b, d);
  }
  __syncthreads();
  if (elem_idx)   // s_el is the element CSR's index array: one coalesced copy
    for (int i = t; i < M * K; i += blockDim.x) elem_idx[i] = s_el[i];
  // ---- a3n + a4: per-node candidates, sorted, adjacent-difference dedupe ----
  if (node_off && !s_big) {
    for (int v = t; v < N; v += blockDim.x) {
      const int b = s_off[v], d = s_off[v + 1] - b;
      uint32_t* seg = raw + (size_t)C * b;
      int m = 0;
      for (int i = 0; i < d; ++i) {
        int row[K];
        const int* r = s_conn + s_el[b + i] * K;
#pragma unroll
        for (int q = 0; q < K; ++q) row[q] = r[q];
        if (simplex) {
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (row[q] != v) seg[m++] = (uint32_t)row[q];
        } else {
          const int p = local_of<T>(row, v);
#pragma unroll
          for (int c = 0; c < C; ++c) seg[m++] = pick<T>(row, nbr_local<T>(p, c));
        }
      }
      int L = 0;
      if (m > kSmallMaxCand) {
        s_big = 1;
      } else if (m <= 16) {
        L = small_sort_unique<16>(seg, m);
      } else if (m <= 32) {
        L = small_sort_unique<32>(seg, m);
      } else {
        small_isort(seg, m);
        for (int i = 0; i < m; ++i)
          if (i == 0 || seg[i] != seg[i - 1]) seg[L++] = seg[i];
      }
      s_ncnt[v] = L;
    }
    __syncthreads();
    if (!s_big) {
      small_block_scan(s_ncnt, N, s_ws);
      for (int v = t; v <= N; v += blockDim.x) node_off[v] = s_ncnt[v];
      for (int v = t; v < N; v += blockDim.x) {
        const uint32_t* seg = raw + (size_t)C * s_off[v];
        const int o = s_ncnt[v], L = s_ncnt[v + 1] - o;
        for (int i = 0; i < L; ++i) fin[o + i] = seg[i];
      }
    }
  }
  __syncthreads();
  if (t == 0) {
    // (read by the host after the stream sync, which makes every write of the kernel visible: no fence)
    ctrl[0] = ERR_NONE;
    ctrl[1] = (node_off && !s_big) ? (unsigned long long)s_ncnt[N] : 0ull;
    ctrl[2] = s_big ? 1ull : 0ull;
  }
}

}  // namespace mn
