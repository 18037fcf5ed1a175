// dist.cuh — the multi-GPU whole path behind mn_find_neighbors_dist (declared in
// include/meshnbr.h).  Included by meshnbr.cu inside namespace mn after dist_bucket_impl /
// dist_finish_impl, which do the per-rank compute; this file holds the exchange protocol and the
// NCCL glue (libnccl.so.2 loaded with dlopen: no link-time NCCL dependency, and inside a PyTorch
// process the NCCL it already loaded is the one used).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

// ------------------------------------------------------------------------------------------------
// NCCL entry points
// ------------------------------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclCommUserRank) comm_user_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag flag;
  std::call_once(flag, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    api.ok = sym(api.get_unique_id, "ncclGetUniqueId") && sym(api.comm_init_rank, "ncclCommInitRank") &&
             sym(api.comm_destroy, "ncclCommDestroy") && sym(api.comm_count, "ncclCommCount") &&
             sym(api.comm_user_rank, "ncclCommUserRank") && sym(api.all_gather, "ncclAllGather") &&
             sym(api.send, "ncclSend") && sym(api.recv, "ncclRecv") && sym(api.group_start, "ncclGroupStart") &&
             sym(api.group_end, "ncclGroupEnd");
  });
  return api;
}

static int nccl_allgather_cb(void* ctx, const void* d_send, void* d_recv, size_t bytes, mn_stream s) {
  const NcclApi& n = nccl();
  if (!n.ok) return 1;
  return n.all_gather(d_send, d_recv, bytes, ncclUint8, (ncclComm_t)ctx, (cudaStream_t)s) == ncclSuccess ? 0 : 1;
}

// All ops of the call in one group: NCCL schedules the sends and receives of every op together.
static int nccl_alltoallv_cb(void* ctx, const mn_a2a_op* ops, int n_ops, mn_stream s) {
  const NcclApi& n = nccl();
  if (!n.ok) return 1;
  ncclComm_t comm = (ncclComm_t)ctx;
  int world = 0;
  if (n.comm_count(comm, &world) != ncclSuccess) return 1;
  if (n.group_start() != ncclSuccess) return 1;
  bool ok = true;
  for (int o = 0; o < n_ops && ok; ++o) {
    const mn_a2a_op& op = ops[o];
    for (int g = 0; g < world && ok; ++g) {
      if (op.send_counts[g] > 0)
        ok = n.send((const char*)op.send + (size_t)op.send_displs[g] * op.elem_bytes,
                    (size_t)op.send_counts[g] * op.elem_bytes, ncclUint8, g, comm, (cudaStream_t)s) == ncclSuccess;
      if (ok && op.recv_counts[g] > 0)
        ok = n.recv((char*)op.recv + (size_t)op.recv_displs[g] * op.elem_bytes,
                    (size_t)op.recv_counts[g] * op.elem_bytes, ncclUint8, g, comm, (cudaStream_t)s) == ncclSuccess;
    }
  }
  const bool ended = n.group_end() == ncclSuccess;
  return ok && ended ? 0 : 1;
}

// ------------------------------------------------------------------------------------------------
// step 2: the exchange plan (host only)
// ------------------------------------------------------------------------------------------------
static mn_status dist_plan(int world, int rank, const int64_t* all, int64_t* rc, int64_t* rr,
                           mn_error_detail* err) {
  const int W = 2 + 2 * world;
  for (int g = 0; g < world; ++g) {
    const int64_t* row = all + (size_t)g * W;
    rc[g] = row[2 + rank];
    rr[g] = row[2 + world + rank];
  }
  for (int g = 0; g < world; ++g) {
    const int64_t stg = all[(size_t)g * W + 1];
    if (stg != MN_OK) return (mn_status)stg;
  }
  uint64_t lowest = ERR_NONE;
  for (int g = 0; g < world; ++g) lowest = std::min(lowest, (uint64_t)all[(size_t)g * W]);
  return decode_err(lowest, err);
}

// ================================================================================================
// Fused bucket-and-send over peer memory (mn_find_neighbors_dist_p2p).  Instead of bucketing into a
// local buffer and then moving the remote buckets with an all-to-all, the owner-digit onesweep pass
// stores every incidence straight into its owner's receive buffer — a symmetric heap each rank
// allocates once and maps into every other rank with CUDA IPC (NVLink peer memory between GPUs;
// the same device in tests) — together with the element row for remote owners.  The transfer
// happens inside the bucketing kernel, tile by tile, while later tiles are still being ranked.
// Needs the count exchange first (the destinations' offsets), and a barrier after the pass.
// ================================================================================================
}  // namespace mn

struct mn_symm {
  mn_comm comm;
  int dev = 0;
  char* local = nullptr;
  size_t cap = 0;
  std::vector<char*> peer;   // peer[g]: rank g's heap mapped here (peer[self] = local)
};

namespace mn {

// (Re)allocate the heap to at least `need` bytes on every rank and exchange the IPC mappings.
// Collective: every rank calls it with the same `need` (derived from the all-gathered counts).
static mn_status symm_reserve(mn_symm* h, size_t need, cudaStream_t s) {
  if (need <= h->cap) return MN_OK;
  const int G = h->comm.world, self = h->comm.rank;
  for (int g = 0; g < G; ++g)
    if (g != self && g < (int)h->peer.size() && h->peer[g]) cudaIpcCloseMemHandle(h->peer[g]);
  if (h->local) cudaFree(h->local);
  h->local = nullptr;
  h->cap = 0;
  h->peer.assign(G, nullptr);
  size_t cap = std::max<size_t>(need + need / 4, (size_t)1 << 20);
  cap = (cap + 4095) & ~(size_t)4095;
  mn_status st = MN_OK;
  char* dbuf = nullptr;
  std::vector<cudaIpcMemHandle_t> all(G);
  cudaIpcMemHandle_t mine{};
  if (cudaMalloc(&h->local, cap) != cudaSuccess) { cudaGetLastError(); h->local = nullptr; st = MN_ERR_OOM; }
  if (st == MN_OK && G > 1 && cudaIpcGetMemHandle(&mine, h->local) != cudaSuccess) { cudaGetLastError(); st = MN_ERR_CUDA; }
  if (G > 1) {   // every rank joins the exchange, failed or not (a zeroed handle marks the failure)
    if (st != MN_OK) std::memset(&mine, 0, sizeof(mine));
    if (cudaMalloc(&dbuf, sizeof(mine) * (G + 1)) != cudaSuccess) { cudaGetLastError(); return MN_ERR_OOM; }
    cudaMemcpyAsync(dbuf, &mine, sizeof(mine), cudaMemcpyHostToDevice, s);
    const int rc = h->comm.allgather(h->comm.ctx, dbuf, dbuf + sizeof(mine), sizeof(mine), (mn_stream)s);
    cudaMemcpyAsync(all.data(), dbuf + sizeof(mine), sizeof(mine) * G, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(dbuf);
    if (rc != 0) return MN_ERR_COMM;
    const cudaIpcMemHandle_t zero{};
    for (int g = 0; g < G; ++g)
      if (std::memcmp(&all[g], &zero, sizeof(zero)) == 0) st = st == MN_OK ? MN_ERR_OOM : st;
    for (int g = 0; g < G && st == MN_OK; ++g) {
      if (g == self) continue;
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, all[g], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        st = MN_ERR_CUDA;
        break;
      }
      h->peer[g] = (char*)p;
    }
  }
  if (st != MN_OK) return st;
  h->peer[self] = h->local;
  h->cap = cap;
  return MN_OK;
}

// Element ids of the received remote incidences (the row table's keys, ascending), skipping the
// own block [own0, own0 + own).
__global__ void __launch_bounds__(256)
k_remote_elems(const uint64_t* __restrict__ pairs, int64_t nr, int64_t own0, int64_t own, int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)(pairs[i < own0 ? i : i + own] & 0xffffffffull);
}

// ================================================================================================
// The multi-GPU path (mn_find_neighbors_dist and _p2p).  One orchestration, two exchanges:
//   1. validation + incidence counts per owner (one read of the shard) and the shard's locality
//      sample, one host read;
//   2. count exchange: one all-gather of [error word, status, counts per owner, locality]; the
//      lowest error of all ranks is returned by every rank;
//   3. bucket-and-send: one owner-digit onesweep pass stores every REMOTE incidence, with its element
//      row, at its place in its owner's receive layout (source-rank order, element-major) — into a
//      local send buffer (then one grouped NCCL all-to-all) or straight into the owner's symmetric
//      heap over peer memory (then an all-gather as a barrier);
//   4. finish: when every shard has locality, the own incidences are never materialised: the
//      element CSR slice is the chunk transpose of (own shard filtered to [lo, hi)) + (received
//      incidences), the node slice the gather with rows from the own shard or the received rows;
//      otherwise the own bucket is written in place between the received ones and the slice built
//      from all of them (stable LSD needs them element-major);
//   5. one all-gather of the slice nnz values.
// ================================================================================================

// Element + node CSR slices of nodes [lo, hi) from the own shard (filtered) and the nr received
// remote incidences (pairs, their rows rr, element ids relems ascending).  Transpose path only.
template <int T>
static mn_status finish_own_conn(const int32_t* conn, int64_t Ms, int64_t base, int64_t own, const uint64_t* rp,
                                 int64_t nr, const int32_t* relems, const int32_t* rr, int64_t lo, int64_t hi,
                                 Mem& mem, mn_csr* node_slice, mn_csr* elem_slice) {
  cudaStream_t s = mem.s;
  mn_status st = MN_OK;
  constexpr int C = Elem<T>::C;
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  const int64_t nloc = hi - lo, n = own + nr;
  const bool aligned = ((uintptr_t)conn & 15) == 0 && ((uintptr_t)rr & 15) == 0;
  std::memset(node_slice, 0, sizeof(*node_slice));
  std::memset(elem_slice, 0, sizeof(*elem_slice));
  int64_t* noff = (int64_t*)mem.get((size_t)(nloc + 1) * 8);
  int64_t* eoff = (int64_t*)mem.get((size_t)(nloc + 1) * 8);
  int32_t* eidx = n ? (int32_t*)mem.get((size_t)n * 4 + 16) : nullptr;
  void* ws = nullptr;
  if (!noff || !eoff || (n && !eidx)) { st = MN_ERR_OOM; goto done; }
  if (n == 0 || nloc == 0) {
    MN_CUDA(cudaMemsetAsync(noff, 0, (size_t)(nloc + 1) * 8, s));
    MN_CUDA(cudaMemsetAsync(eoff, 0, (size_t)(nloc + 1) * 8, s));
    MN_CUDA(cudaStreamSynchronize(s));
  } else {
    const int64_t nch = tiles_of(nloc, kChunkNodes);
    Arena ar;
    unsigned long long* errw = ar.take<unsigned long long>(2);
    uint32_t* tickets = ar.take<uint32_t>(8);
    unsigned int* ngiant = ar.take<unsigned int>(1);
    unsigned int* nsgiant = ar.take<unsigned int>(1);
    unsigned int* ovf = ar.take<unsigned int>(1);
    uint64_t* sstatus = ar.take<uint64_t>((size_t)tiles_of(nloc, kScanTile) + 1);
    int32_t* ccur = ar.take<int32_t>((size_t)nch + 1);    // fixed-bucket cursors
    int32_t* ccnt = ar.take<int32_t>((size_t)nch + 1);    // fallback counts
    int32_t* cnt = ar.take<int32_t>((size_t)nloc + 1);
    int32_t* lofs = ar.take<int32_t>((size_t)nloc + 1);
    const size_t head = ar.off;
    int64_t* cbase = ar.take<int64_t>((size_t)nch + 1);
    uint32_t* temp = ar.take<uint32_t>((size_t)std::max<int64_t>(C * n, 2 * n + 64));   // buckets, then node lists
    uint8_t* bnode = ar.take<uint8_t>((size_t)2 * n + 64);
    uint32_t* giants = ar.take<uint32_t>((size_t)nloc + 1);
    uint32_t* sgiants = ar.take<uint32_t>((size_t)nloc + 1);
    const int64_t ngn = tiles_of(nloc, kNodeThreads);         // node chunks of the gather
    int32_t* ncsum = ar.take<int32_t>((size_t)ngn + 1);         // their list totals
    int64_t* ncb = ar.take<int64_t>((size_t)ngn + 1);           // and bases
    ws = mem.get(ar.off);
    if (!ws) { st = MN_ERR_OOM; goto done; }
    {
      char* bb = (char*)ws;
      auto fix = [&](auto* q) { return (decltype(q))(bb + (size_t)q); };
      errw = fix(errw); tickets = fix(tickets); ngiant = fix(ngiant); nsgiant = fix(nsgiant); ovf = fix(ovf);
      sstatus = fix(sstatus); ccur = fix(ccur); ccnt = fix(ccnt); cnt = fix(cnt); lofs = fix(lofs);
      cbase = fix(cbase); temp = fix(temp); bnode = fix(bnode); giants = fix(giants); sgiants = fix(sgiants);
      ncsum = fix(ncsum); ncb = fix(ncb);
      int32_t* belem = reinterpret_cast<int32_t*>(temp);
      MN_CUDA(cudaMemsetAsync(ws, 0, head, s));
      MN_CUDA(cudaMemsetAsync(errw, 0xFF, 8, s));
      int64_t capl = (2 * n / nch) & ~(int64_t)31;
      const int ovr = g_chunk_cap.load();
      if (ovr > 0 && ovr < capl) capl = ovr;
      if (capl > (int64_t)INT32_MAX - 4096) capl = (int64_t)INT32_MAX - 4096;
      const int cap = (int)capl;
      const PairSrc ps = pair_src(rp, nr);
      // element CSR slice: own shard (range-filtered) + received incidences into the same fixed
      // chunk buckets; the guarded counted fallback replaces them when a bucket overflows
      MN_CUDA(launch("elem_scatter", 4.0 * Elem<T>::K * Ms + 5.0 * own, s, [&] {
        if (aligned)
          k_chunk_scatter_fixed<T, true, 1, true><<<hist_grid(Ms), 256, 0, s>>>(conn, Ms, INT32_MAX, cap, ccur, belem,
                                                                            bnode, errw, ovf, lo, hi, base);
        else
          k_chunk_scatter_fixed<T, false, 1, true><<<hist_grid(Ms), 256, 0, s>>>(conn, Ms, INT32_MAX, cap, ccur,
                                                                             belem, bnode, errw, ovf, lo, hi, base);
      }));
      if (nr > 0)
        MN_CUDA(launch("elem_scatter", 13.0 * nr, s, [&] {
          k_pairs_chunk_scatter<true><<<stream_grid(nr), 256, 0, s>>>(ps, nr, lo, cap, nullptr, ccur, belem, bnode,
                                                                      ovf);
        }));
      MN_CUDA(launch("scan_counts", 12.0 * nch, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch, kScanTile), kScanThreads, 0, s>>>(
            ccur, nch, cbase, sstatus, tickets + 0, 1);
      }));
      MN_CUDA(launch("count_fallback", 0.0, s, [&] {
        if (aligned)
          k_chunk_count<T, true, true><<<count_grid(Ms), 256, 0, s>>>(conn, Ms, INT32_MAX, ccnt, errw, lo, hi, ovf);
        else
          k_chunk_count<T, false, true><<<count_grid(Ms), 256, 0, s>>>(conn, Ms, INT32_MAX, ccnt, errw, lo, hi, ovf);
        if (nr > 0) k_pairs_chunk_count<<<stream_grid(nr), 256, 0, s>>>(ps, nr, lo, ccnt, ovf);
      }));
      MN_CUDA(launch("scan_fallback", 0.0, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(nch, kScanTile), kScanThreads, 0, s>>>(
            ccnt, nch, cbase, sstatus, tickets + 1, 2, ovf);
      }));
      MN_CUDA(launch("scatter_fallback", 0.0, s, [&] {
        if (aligned)
          k_chunk_scatter<T, true, true><<<hist_grid(Ms), 256, 0, s>>>(conn, Ms, cbase, lofs, belem, bnode, errw, lo,
                                                                      hi, ovf, base);
        else
          k_chunk_scatter<T, false, true><<<hist_grid(Ms), 256, 0, s>>>(conn, Ms, cbase, lofs, belem, bnode, errw,
                                                                       lo, hi, ovf, base);
        if (nr > 0)
          k_pairs_chunk_scatter<false><<<stream_grid(nr), 256, 0, s>>>(ps, nr, lo, 0, cbase, lofs, belem, bnode, ovf);
      }));
      MN_CUDA(launch("elem_segsort", 9.0 * n + 8.0 * (nloc + 1), s, [&] {
        k_chunk_sort<true><<<(unsigned)nch, kChunkNodes, 0, s>>>(cbase, nloc, belem, bnode, eoff, eidx, sgiants,
                                                                  nsgiant, errw, ovf, cap);
      }));
      const int scap = 48 * 1024;
      cudaFuncSetAttribute(k_segsort_giant, cudaFuncAttributeMaxDynamicSharedMemorySize, scap * 4);
      MN_CUDA(launch("segsort_giant", 0.0, s, [&] {
        k_segsort_giant<<<148, 1024, scap * 4, s>>>(eoff, eidx, sgiants, nsgiant, scap, errw);
      }));
      MN_CUDA(cudaMemsetAsync(lofs, 0, (size_t)(nloc + 1) * 4, s));
      // node CSR slice: rows of own elements from the shard, of remote ones from the received table
      const RowSrc rs{conn, base, Ms, relems, rr, nr};
      const unsigned ng = (unsigned)tiles_of(nloc, kNodeThreads);
      MN_CUDA(launch("node_gather", 8.0 * (nloc + 1) + 4.0 * n + 4.0 * Elem<T>::K * (Ms + nr) + 8.0 * nloc, s, [&] {
        if (aligned)
          k_node_gather_t<T, true, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, nloc, temp, cnt, lofs, giants,
                                                                     ngiant, errw, lo, ncsum);
        else
          k_node_gather_t<T, false, true><<<ng, kNodeThreads, 0, s>>>(eoff, eidx, rs, nloc, temp, cnt, lofs, giants,
                                                                      ngiant, errw, lo, ncsum);
      }));
      const int cap2 = 48 * 1024;
      static PerDevice attr;
      attr.once([&] {
        cudaFuncSetAttribute(k_node_giant<T, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap2 * 4);
        cudaFuncSetAttribute(k_node_giant<T, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap2 * 4);
        return 0;
      });
      MN_CUDA(launch("node_giant", 0.0, s, [&] {
        if (aligned)
          k_node_giant<T, true, true><<<148, 1024, cap2 * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant, cap2,
                                                                 errw, lo, ncsum);
        else
          k_node_giant<T, false, true><<<148, 1024, cap2 * 4, s>>>(eoff, eidx, rs, temp, cnt, lofs, giants, ngiant,
                                                                  cap2, errw, lo, ncsum);
      }));
      // node offsets as in the 1-GPU path: scan of the chunk totals, offsets written by the compaction
      MN_CUDA(launch("scan_counts", 12.0 * ngn, s, [&] {
        k_scan_i32<kScanThreads, kScanItems><<<(unsigned)tiles_of(ngn, kScanTile), kScanThreads, 0, s>>>(
            ncsum, ngn, ncb, sstatus, tickets + 2, 3);
      }));
      MN_CUDA(read_words(host + 1, ncb + ngn, 8, s));
      MN_CUDA(cudaStreamSynchronize(s));
      const int64_t U = (int64_t)host[1];
      prof_add_bytes("node_gather", 4.0 * U);
      if (U) {
        node_slice->indices = (int32_t*)mem.get((size_t)U * 4);
        if (!node_slice->indices) { st = MN_ERR_OOM; goto done; }
      }
      MN_CUDA(launch("node_compact", 8.0 * U + 24.0 * nloc, s, [&] {
        k_node_compact_cb<<<(unsigned)ngn, kNodeThreads, 0, s>>>(eoff, C, temp, lofs, cnt, ncb, nloc, noff,
                                                                 node_slice->indices);
      }));
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

template <int T, int BINS>
static mn_status dist2_impl(const int32_t* conn, int64_t M, int64_t base, int64_t N, const mn_comm* comm, mn_symm* h,
                            Mem& mem, mn_csr* node_slice, mn_csr* elem_slice, mn_dist_info* info,
                            mn_error_detail* err) {
  constexpr int K = Elem<T>::K;
  cudaStream_t s = mem.s;
  const bool p2p = h != nullptr;
  const int G = comm->world, self = comm->rank;
  const int W = 2 + 2 * G;
  const Plan P = make_plan(T, M, N);
  const int64_t Pe = P.Pe;
  mn_status st = MN_OK, local = MN_OK;
  std::memset(node_slice, 0, sizeof(*node_slice));
  std::memset(elem_slice, 0, sizeof(*elem_slice));
  uint64_t* host = pinned_pair();
  if (!host) return MN_ERR_CUDA;
  const uint64_t chunk = (uint64_t)((N + G - 1) / G > 0 ? (N + G - 1) / G : 1);
  const int64_t lo = std::min<int64_t>(N, (int64_t)chunk * self), hi = std::min<int64_t>(N, (int64_t)chunk * (self + 1));
  std::vector<int64_t> row((size_t)W, 0), all((size_t)W * G, 0), rc(G, 0), rr(G, 0), nnz_all((size_t)2 * G, 0);
  std::vector<unsigned long long> hh(BINS, 0);
  std::vector<uint64_t*> dsth(G, nullptr);
  std::vector<int32_t*> rowh(G, nullptr);
  std::vector<int64_t> sc(G, 0), sd(G, 0), rcn(G, 0), rd(G, 0), sdr(G, 0), rdr(G, 0);
  int64_t nnz2[2] = {0, 0};
  uint64_t ew = ERR_NONE;
  bool all_local = false;
  int64_t in = 0, own = 0, own0 = 0, nr = 0;
  uint64_t *sendp = nullptr, *recvp = nullptr;
  int32_t *sendr = nullptr, *recvr = nullptr, *relems = nullptr;
  const uint64_t* rpairs = nullptr;   // the received (and, without locality, own) incidences
  const int32_t* rrows = nullptr;
  int64_t* dx = (int64_t*)mem.get((size_t)W * (G + 1) * 8 + (size_t)G * 16);
  if (!dx) return MN_ERR_OOM;
  void** dptr = (void**)(dx + (size_t)W * (G + 1));
  const int64_t tiles = tiles_of(Pe, kTile);
  Arena ar;
  unsigned long long* errw = ar.take<unsigned long long>(2);
  unsigned long long* smp = ar.take<unsigned long long>(2);
  uint32_t* tickets = ar.take<uint32_t>(8);
  unsigned long long* hist = ar.take<unsigned long long>(BINS);
  unsigned long long* hist2 = ar.take<unsigned long long>(BINS);
  uint64_t* bases = ar.take<uint64_t>(BINS);
  uint64_t* status = ar.take<uint64_t>((size_t)(tiles ? tiles : 1) * BINS);
  unsigned long long* dnrem = ar.take<unsigned long long>(1);
  const size_t head = ar.off;
  char* ws = (char*)mem.get(ar.off);
  bool loc = false;        // this shard's locality (the element algorithm of the 1-GPU path)
  int64_t nrem = 0;        // remote incidences of this shard
  uint64_t* rem = nullptr;   // (coherent shards) the remote incidences in element order
  if (!ws) local = MN_ERR_OOM;
  if (local == MN_OK) {
    errw = (unsigned long long*)(ws + (size_t)errw); smp = (unsigned long long*)(ws + (size_t)smp);
    tickets = (uint32_t*)(ws + (size_t)tickets); hist = (unsigned long long*)(ws + (size_t)hist);
    hist2 = (unsigned long long*)(ws + (size_t)hist2);
    bases = (uint64_t*)(ws + (size_t)bases); status = (uint64_t*)(ws + (size_t)status);
    dnrem = (unsigned long long*)(ws + (size_t)dnrem);
    const bool aligned = ((uintptr_t)conn & 15) == 0;
    if (cudaMemsetAsync(ws, 0, head, s) != cudaSuccess || cudaMemsetAsync(errw, 0xFF, 8, s) != cudaSuccess)
      local = MN_ERR_CUDA;
    // ---- 0. locality of the shard (decides whether the remote incidences are compacted) ----
    const int mode = g_elem_path.load();
    if (local == MN_OK && M > 0 && mode == 0) {
      if (launch("locality_sample", 0.0, s, [&] {
            if (aligned) k_locality_sample<T, true><<<64, 256, 0, s>>>(conn, M, smp);
            else k_locality_sample<T, false><<<64, 256, 0, s>>>(conn, M, smp);
          }) != cudaSuccess ||
          read_words(host + 2, smp, 16, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        local = MN_ERR_CUDA;
    }
    loc = M == 0 || mode == 2 ||
          (mode == 0 && local == MN_OK && host[3] > 0 && (double)host[2] < kTransposeMaxGroupRatio * (double)host[3]);
    if (loc && M > 0 && local == MN_OK) {
      rem = (uint64_t*)mem.get((size_t)Pe * 8);
      if (!rem) local = MN_ERR_OOM;
    }
    // ---- 1. validation + incidence counts per owner (+ the remote incidences), one host read ----
    if (local == MN_OK && M > 0) {
      cudaError_t e;
      if (rem)
        e = launch("hist_remote", 4.0 * P.K * M, s, [&] {
          if (aligned)
            k_hist_remote<T, BINS, true><<<hist_grid(M), 256, 0, s>>>(conn, M, N, base, chunk, G, self, hist, errw,
                                                                        rem, dnrem);
          else
            k_hist_remote<T, BINS, false><<<hist_grid(M), 256, 0, s>>>(conn, M, N, base, chunk, G, self, hist, errw,
                                                                         rem, dnrem);
        });
      else
        e = launch("hist_validate", 4.0 * P.K * M, s, [&] {
          k_hist_validate<T, BINS, false><<<hist_grid(M), 256, 0, s>>>(conn, M, N, base, P.dp, 1, chunk, hist, errw);
        });
      if (e != cudaSuccess) local = MN_ERR_CUDA;
    }
    if (local == MN_OK &&
        (cudaMemcpyAsync(hh.data(), hist, BINS * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
         read_words(host, errw, 8, s) != cudaSuccess ||
         cudaStreamSynchronize(s) != cudaSuccess))
      local = MN_ERR_CUDA;
    if (local == MN_OK) ew = host[0];
    for (int g = 0; g < G; ++g)
      if (g != self) nrem += (int64_t)hh[g];
  }
  // ---- 2. count exchange: [error word, status, counts per owner, locality flag] ----
  row[0] = (int64_t)ew;
  row[1] = local;
  if (local == MN_OK && ew == ERR_NONE)
    for (int g = 0; g < G; ++g) row[2 + g] = (int64_t)hh[g];
  row[2 + G] = (local == MN_OK && loc) ? 1 : 0;
  MN_CUDA(cudaMemcpyAsync(dx, row.data(), (size_t)W * 8, cudaMemcpyHostToDevice, s));
  if (comm->allgather(comm->ctx, dx, dx + W, (size_t)W * 8, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  MN_CUDA(cudaMemcpyAsync(all.data(), dx + W, (size_t)W * G * 8, cudaMemcpyDeviceToHost, s));
  MN_CUDA(cudaStreamSynchronize(s));
  st = dist_plan(G, self, all.data(), rc.data(), rr.data(), err);
  if (st != MN_OK) goto done;
  all_local = true;
  for (int g = 0; g < G; ++g) all_local = all_local && all[(size_t)g * W + 2 + G] != 0;
  // ---- 3. receive layouts (source-rank order; the own block only without locality) ----
  {
    auto cnt = [&](int r, int g) { return all[(size_t)r * W + 2 + g]; };
    auto pbytes = [](int64_t n) { return ((size_t)n * 8 + 255) & ~(size_t)255; };
    std::vector<int64_t> ing(G, 0), offp(G, 0), offr(G, 0);
    size_t need = 0;
    for (int g = 0; g < G; ++g) {
      for (int r = 0; r < G; ++r)
        if (r != g || !all_local) ing[g] += cnt(r, g);
      const int64_t remote_in = ing[g] - (all_local ? 0 : cnt(g, g));
      need = std::max(need, pbytes(ing[g]) + (size_t)remote_in * 4 * K + 256);
      for (int r = 0; r < self; ++r)
        if (r != g || !all_local) offp[g] += cnt(r, g);
      // rows: remote sources only; sources after g skip g's own block (present without locality)
      offr[g] = offp[g] - (!all_local && self > g ? cnt(g, g) : 0);
    }
    in = ing[self];
    own = cnt(self, self);
    own0 = all_local ? 0 : offp[self];
    nr = in - (all_local ? 0 : own);
    if (p2p) {
      st = symm_reserve(h, need, s);
      if (st != MN_OK) goto done;
      for (int g = 0; g < G; ++g) {
        dsth[g] = (g == self && all_local) ? nullptr : reinterpret_cast<uint64_t*>(h->peer[g]) + offp[g];
        rowh[g] = g == self ? nullptr : reinterpret_cast<int32_t*>(h->peer[g] + pbytes(ing[g])) + offr[g] * K;
      }
      rpairs = reinterpret_cast<const uint64_t*>(h->local);
      rrows = reinterpret_cast<const int32_t*>(h->local + pbytes(in));
    } else {
      // local send buffers (remote buckets in rank order), receive buffers in source-rank order
      int64_t ns = 0;
      for (int g = 0; g < G; ++g)
        if (g != self) ns += cnt(self, g);
      sendp = ns ? (uint64_t*)mem.get((size_t)ns * 8) : nullptr;
      sendr = ns ? (int32_t*)mem.get((size_t)ns * 4 * K) : nullptr;
      recvp = in ? (uint64_t*)mem.get((size_t)in * 8) : nullptr;
      recvr = nr ? (int32_t*)mem.get((size_t)nr * 4 * K) : nullptr;
      if ((ns && (!sendp || !sendr)) || (in && !recvp) || (nr && !recvr)) { st = MN_ERR_OOM; goto done; }
      int64_t a = 0, b = 0, c = 0;
      for (int g = 0; g < G; ++g) {
        if (g == self) {
          dsth[g] = all_local ? nullptr : recvp + own0;   // own bucket in place (no exchange)
        } else {
          dsth[g] = sendp + a;
          rowh[g] = sendr + a * K;
          sd[g] = a;
          sc[g] = cnt(self, g);
          a += sc[g];
        }
        rd[g] = b;   // pairs received from g (own block skipped: not exchanged)
        rcn[g] = g == self ? 0 : cnt(g, self);
        b += (g == self) ? (all_local ? 0 : own) : rcn[g];
        rdr[g] = c;
        c += rcn[g];
      }
      rpairs = recvp;
      rrows = recvr;
    }
  }
  // ---- 4. bucket-and-send: one onesweep pass over the shard's incidences ----
  MN_CUDA(cudaMemcpyAsync(dptr, dsth.data(), (size_t)G * 8, cudaMemcpyHostToDevice, s));
  MN_CUDA(cudaMemcpyAsync(dptr + G, rowh.data(), (size_t)G * 8, cudaMemcpyHostToDevice, s));
  if (M > 0 && all_local && nrem > 0) {
    // only the remote incidences (appended by pass 1) are put in element order, bucketed and sent
    {
      uint32_t* rk = (uint32_t*)mem.get((size_t)nrem * 8);
      if (!rk) { st = MN_ERR_OOM; goto done; }
      uint32_t* rv = rk + nrem;
      MN_CUDA(launch("remote_order", 16.0 * nrem, s, [&] {
        k_split_pairs<<<stream_grid(nrem), 256, 0, s>>>(rem, nrem, base, rk, rv);
      }));
      st = lsd_sort<uint32_t, true>(rk, rv, nrem, node_bits(M), mem);
      if (st == MN_OK)
        MN_CUDA(launch("remote_order", 16.0 * nrem, s, [&] {
          k_join_pairs<<<stream_grid(nrem), 256, 0, s>>>(rk, rv, nrem, base, rem);
        }));
      mem.put(rk);
      if (st != MN_OK) goto done;
    }
    MN_CUDA(cudaMemcpyAsync(hist2, hist, BINS * 8, cudaMemcpyDeviceToDevice, s));
    MN_CUDA(cudaMemsetAsync(hist2 + self, 0, 8, s));
    BasesDesc bd{};
    bd.npass = 1;
    bd.hidx[0] = 0;
    bd.mult[0] = 1;
    MN_CUDA(launch("bucket_bases", 0.0, s, [&] { k_bucket_bases<BINS><<<1, BINS, 0, s>>>(hist2, bd, bases, errw); }));
    PassArgs pe{};
    pe.keys_in = rem; pe.conn = conn; pe.elem_base = base; pe.n = nrem;
    pe.pd.shift = 32; pe.pd.div = chunk; pe.pd.mask = 0;
    pe.bases = bases; pe.status = status; pe.ticket = tickets; pe.epoch = 1; pe.err = errw;
    pe.dst = (uint64_t* const*)dptr;
    pe.rowdst = (int32_t* const*)(dptr + G);
    pe.self = self;
    using Sm = OnesweepSmem<kPassThreads, kPassItems, BINS>;
    const size_t smem = ((sizeof(Sm) + 15) & ~size_t(15)) + (size_t)kTile * 8;
    auto kern = k_onesweep<uint64_t, 0, T, false, true, BINS, kPassThreads, kPassItems, kPassWindow, kPassMinBlocks,
                           0, false, false, true>;
    static PerDevice attr0;
    attr0.once([&] {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      return 0;
    });
    MN_CUDA(launch(p2p ? "bucket_send_p2p" : "bucket_send", (16.0 + 4.0 * K) * nrem, s, [&] {
      kern<<<(unsigned)tiles_of(nrem, kTile), kPassThreads, smem, s>>>(pe);
    }));
  } else if (M > 0 && !all_local) {
    BasesDesc bd{};
    bd.npass = 1;
    bd.hidx[0] = 0;
    bd.mult[0] = 1;
    MN_CUDA(launch("bucket_bases", 0.0, s, [&] { k_bucket_bases<BINS><<<1, BINS, 0, s>>>(hist, bd, bases, errw); }));
    PassArgs pe{};
    pe.conn = conn; pe.elem_base = base; pe.n = Pe;
    pe.pd.shift = 32; pe.pd.div = chunk; pe.pd.mask = 0;
    pe.bases = bases; pe.status = status; pe.ticket = tickets; pe.epoch = 1; pe.err = errw;
    pe.dst = (uint64_t* const*)dptr;
    pe.rowdst = (int32_t* const*)(dptr + G);
    pe.self = self;
    using Sm = OnesweepSmem<kPassThreads, kPassItems, BINS>;
    const size_t smem = ((sizeof(Sm) + 15) & ~size_t(15)) + (size_t)kTile * 8;
    auto kern = k_onesweep<uint64_t, 3, T, false, true, BINS, kPassThreads, kPassItems, kPassWindow, kPassMinBlocks,
                           0, false, false, true>;
    static PerDevice attr;
    attr.once([&] {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      return 0;
    });
    MN_CUDA(launch(p2p ? "bucket_send_p2p" : "bucket_send", 4.0 * Pe + 8.0 * Pe, s, [&] {
      kern<<<(unsigned)tiles, kPassThreads, smem, s>>>(pe);
    }));
  }
  // ---- 5. the exchange ----
  if (p2p) {   // barrier: every rank's stores into this heap are complete past this all-gather
    MN_CUDA(cudaMemcpyAsync(dx, nnz2, 8, cudaMemcpyHostToDevice, s));
    if (comm->allgather(comm->ctx, dx, dx + 2, 8, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  } else {
    std::vector<int64_t> scr(G, 0);
    for (int g = 0; g < G; ++g) scr[g] = g == self ? 0 : sc[g];
    const mn_a2a_op ops[2] = {
        {sendp, scr.data(), sd.data(), recvp, rcn.data(), rd.data(), 8},
        {sendr, scr.data(), sd.data(), recvr, rcn.data(), rdr.data(), (size_t)K * 4},
    };
    if (comm->alltoallv(comm->ctx, ops, 2, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
    mem.put(sendp); sendp = nullptr;
    mem.put(sendr); sendr = nullptr;
  }
  if (info) {
    int64_t sent = 0, got = 0;
    for (int g = 0; g < G; ++g)
      if (g != self) {
        sent += all[(size_t)self * W + 2 + g] * (8 + 4 * K);
        got += all[(size_t)g * W + 2 + self] * (8 + 4 * K);
      }
    info->sent_bytes = sent;
    info->recv_bytes = got;
    info->own_incidences = own;
  }
  // ---- 6. finish ----
  if (nr > 0) {
    relems = (int32_t*)mem.get((size_t)nr * 4);
    if (!relems) { st = MN_ERR_OOM; goto done; }
    MN_CUDA(launch("remote_elems", 12.0 * nr, s, [&] {
      k_remote_elems<<<stream_grid(nr), 256, 0, s>>>(rpairs, nr, all_local ? nr : own0, all_local ? 0 : own, relems);
    }));
  }
  if (all_local) {
    st = finish_own_conn<T>(conn, M, base, own, rpairs, nr, relems, rrows, lo, hi, mem, node_slice, elem_slice);
  } else {
    if (in > INT32_MAX) { st = MN_ERR_CAPACITY; goto done; }
    st = dist_finish_impl<T>(pair_src(rpairs, in), in, relems, rrows, nr, conn, base, M, N, lo, hi, mem, node_slice,
                             elem_slice);
  }
  if (st != MN_OK) goto done;
  mem.put(relems); relems = nullptr;
  mem.put(recvp); recvp = nullptr;
  mem.put(recvr); recvr = nullptr;
  mem.put(rem); rem = nullptr;
  // ---- 7. global offset bases ----
  nnz2[0] = node_slice->nnz;
  nnz2[1] = elem_slice->nnz;
  MN_CUDA(cudaMemcpyAsync(dx, nnz2, 16, cudaMemcpyHostToDevice, s));
  if (comm->allgather(comm->ctx, dx, dx + 2, 16, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  MN_CUDA(cudaMemcpyAsync(nnz_all.data(), dx + 2, (size_t)16 * G, cudaMemcpyDeviceToHost, s));
  MN_CUDA(cudaStreamSynchronize(s));
  mem.put(ws);
  mem.put(dx);
  if (info) {
    info->lo = lo;
    info->hi = hi;
    info->node_base = info->elem_base = info->node_nnz_total = info->elem_nnz_total = 0;
    for (int g = 0; g < G; ++g) {
      if (g < self) { info->node_base += nnz_all[2 * g]; info->elem_base += nnz_all[2 * g + 1]; }
      info->node_nnz_total += nnz_all[2 * g];
      info->elem_nnz_total += nnz_all[2 * g + 1];
    }
  }
  return MN_OK;
done:
  cudaStreamSynchronize(s);
  mem.put(ws);
  mem.put(dx);
  mem.put(sendp);
  mem.put(sendr);
  mem.put(recvp);
  mem.put(recvr);
  mem.put(relems);
  mem.put(rem);
  mn_csr_release(node_slice, (mn_stream)s);
  mn_csr_release(elem_slice, (mn_stream)s);
  return st;
}

static mn_status dist2_dispatch(mn_elem_type t, const int32_t* conn, int64_t M, int64_t base, int64_t N,
                                const mn_comm* comm, mn_symm* h, Mem& mem, mn_csr* ns, mn_csr* es, mn_dist_info* info,
                                mn_error_detail* err) {
  const bool b512 = comm->world > 256;
#define MN_D2(TT) \
  return b512 ? dist2_impl<TT, 512>(conn, M, base, N, comm, h, mem, ns, es, info, err) \
              : dist2_impl<TT, 256>(conn, M, base, N, comm, h, mem, ns, es, info, err)
  switch (t) {
    case MN_TRI3: MN_D2(MN_TRI3);
    case MN_QUAD4: MN_D2(MN_QUAD4);
    case MN_TET4: MN_D2(MN_TET4);
    default: MN_D2(MN_HEX8);
  }
#undef MN_D2
}
