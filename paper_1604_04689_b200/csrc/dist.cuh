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

// ------------------------------------------------------------------------------------------------
// the whole call
// ------------------------------------------------------------------------------------------------
template <int T>
static mn_status dist_impl(const int32_t* conn, int64_t M, int64_t base, int64_t N, const mn_comm* comm, Mem& mem,
                           mn_csr* node_slice, mn_csr* elem_slice, mn_dist_info* info, mn_error_detail* err) {
  constexpr int K = Elem<T>::K;
  cudaStream_t s = mem.s;
  const int G = comm->world, self = comm->rank;
  const int W = 2 + 2 * G;
  const int64_t Pe = M * K;
  mn_status st = MN_OK, local = MN_OK;
  std::memset(node_slice, 0, sizeof(*node_slice));
  std::memset(elem_slice, 0, sizeof(*elem_slice));
  std::vector<int64_t> hc(G, 0), hrc(G, 0), rc(G, 0), rr(G, 0), row((size_t)W, 0), all((size_t)W * G, 0);
  uint64_t ew = ERR_NONE;
  int32_t *relems = nullptr, *rrows = nullptr;
  uint64_t* pairs = nullptr;
  uint64_t *recv_pairs = nullptr;
  int32_t *recv_elems = nullptr, *recv_rows = nullptr;
  int64_t* dx = nullptr;   // device staging of the all-gathers
  int64_t lo = 0, hi = 0, before = 0, after = 0, nr = 0, own = 0;
  std::vector<int64_t> sd(G, 0), rd(G, 0), sdr(G, 0), rdr(G, 0), sc(G, 0), rcz(G, 0);
  int64_t nnz2[2] = {0, 0};
  std::vector<int64_t> nnz_all((size_t)2 * G, 0);
  const uint64_t chunk = (uint64_t)((N + G - 1) / G > 0 ? (N + G - 1) / G : 1);
  lo = std::min<int64_t>(N, (int64_t)chunk * self);
  hi = std::min<int64_t>(N, (int64_t)chunk * (self + 1));

  // the all-gather staging first: past this point every failure still joins the count exchange
  dx = (int64_t*)mem.get((size_t)W * (G + 1) * 8);
  if (!dx) return MN_ERR_OOM;
  // ---- 1. validate + bucket (a local failure is carried into the count exchange) ----
  if (Pe > 0) {
    pairs = (uint64_t*)mem.get((size_t)Pe * 8);
    if (!pairs) local = MN_ERR_OOM;
  }
  if (local == MN_OK) {
    local = (G <= 256 ? dist_bucket_impl<T, 256> : dist_bucket_impl<T, 512>)(
        conn, M, base, N, G, self, pairs, hc.data(), &relems, &rrows, hrc.data(), mem, err, &ew);
  }
  if (local != MN_OK) {
    std::fill(hc.begin(), hc.end(), 0);
    std::fill(hrc.begin(), hrc.end(), 0);
  }
  // ---- 2. count exchange: one all-gather of [error word, status, counts, row counts] ----
  row[0] = (int64_t)ew;
  row[1] = local;
  for (int g = 0; g < G; ++g) { row[2 + g] = hc[g]; row[2 + G + g] = hrc[g]; }
  MN_CUDA(cudaMemcpyAsync(dx, row.data(), (size_t)W * 8, cudaMemcpyHostToDevice, s));
  if (comm->allgather(comm->ctx, dx, dx + W, (size_t)W * 8, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  MN_CUDA(cudaMemcpyAsync(all.data(), dx + W, (size_t)W * G * 8, cudaMemcpyDeviceToHost, s));
  MN_CUDA(cudaStreamSynchronize(s));
  st = dist_plan(G, self, all.data(), rc.data(), rr.data(), err);
  if (st != MN_OK) goto done;

  // ---- 3. payload exchange: remote incidences, remote element ids, their rows ----
  for (int g = 0; g < G; ++g) {
    if (g < self) before += rc[g];
    if (g > self) after += rc[g];
    if (g != self) nr += rr[g];
  }
  own = rc[self];
  {
    int64_t a = 0, b = 0, c = 0, d = 0;
    for (int g = 0; g < G; ++g) {
      sd[g] = a; a += hc[g];                  // pairs: bucket g starts at the prefix of the counts
      sc[g] = g == self ? 0 : hc[g];
      rd[g] = b; if (g != self) b += rc[g];   // received pairs packed without the own bucket
      rcz[g] = g == self ? 0 : rc[g];
      sdr[g] = c; c += hrc[g];                // rows: grouped by destination (none for self)
      rdr[g] = d; d += g == self ? 0 : rr[g];
    }
  }
  if (before + after > 0) {
    recv_pairs = (uint64_t*)mem.get((size_t)(before + after) * 8);
    if (!recv_pairs) { st = MN_ERR_OOM; goto done; }
  }
  if (nr > 0) {
    recv_elems = (int32_t*)mem.get((size_t)nr * 4);
    recv_rows = (int32_t*)mem.get((size_t)nr * K * 4);
    if (!recv_elems || !recv_rows) { st = MN_ERR_OOM; goto done; }
  }
  {
    std::vector<int64_t> rrz(G);
    for (int g = 0; g < G; ++g) rrz[g] = g == self ? 0 : rr[g];
    const mn_a2a_op ops[3] = {
        {pairs, sc.data(), sd.data(), recv_pairs, rcz.data(), rd.data(), 8},
        {relems, hrc.data(), sdr.data(), recv_elems, rrz.data(), rdr.data(), 4},
        {rrows, hrc.data(), sdr.data(), recv_rows, rrz.data(), rdr.data(), (size_t)K * 4},
    };
    if (comm->alltoallv(comm->ctx, ops, 3, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  }
  if (info) {
    int64_t sent = 0, got = 0;
    for (int g = 0; g < G; ++g)
      if (g != self) {
        sent += hc[g] * 8 + hrc[g] * 4 * (K + 1);
        got += rc[g] * 8 + rr[g] * 4 * (K + 1);
      }
    info->sent_bytes = sent;
    info->recv_bytes = got;
    info->own_incidences = own;
  }

  // ---- 4. local finish over (lower ranks' pairs, own bucket in place, higher ranks' pairs) ----
  {
    const uint64_t* ownp = pairs ? pairs + sd[self] : recv_pairs;
    const PairSrc ps{{recv_pairs, ownp, recv_pairs ? recv_pairs + before : ownp},
                     {before, before + own, before + own + after}};
    const int64_t n = before + own + after;
    if (n > INT32_MAX) { st = MN_ERR_CAPACITY; goto done; }
    st = dist_finish_impl<T>(ps, n, recv_elems, recv_rows, nr, conn, base, M, N, lo, hi, mem, node_slice, elem_slice);
    if (st != MN_OK) goto done;
  }
  mem.put(pairs); pairs = nullptr;
  mem.put(recv_pairs); recv_pairs = nullptr;
  mem.put(recv_elems); recv_elems = nullptr;
  mem.put(recv_rows); recv_rows = nullptr;
  mem.put(relems); relems = nullptr;
  mem.put(rrows); rrows = nullptr;

  // ---- 5. global offset bases: all-gather of the slice nnz values ----
  nnz2[0] = node_slice->nnz;
  nnz2[1] = elem_slice->nnz;
  MN_CUDA(cudaMemcpyAsync(dx, nnz2, 16, cudaMemcpyHostToDevice, s));
  if (comm->allgather(comm->ctx, dx, dx + 2, 16, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  MN_CUDA(cudaMemcpyAsync(nnz_all.data(), dx + 2, (size_t)16 * G, cudaMemcpyDeviceToHost, s));
  MN_CUDA(cudaStreamSynchronize(s));
  mem.put(dx); dx = nullptr;
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
  mem.put(pairs);
  mem.put(recv_pairs);
  mem.put(recv_elems);
  mem.put(recv_rows);
  mem.put(relems);
  mem.put(rrows);
  mem.put(dx);
  mn_csr_release(node_slice, (mn_stream)s);
  mn_csr_release(elem_slice, (mn_stream)s);
  return st;
}

static mn_status dist_dispatch(mn_elem_type t, const int32_t* conn, int64_t M, int64_t base, int64_t N,
                               const mn_comm* comm, Mem& mem, mn_csr* ns, mn_csr* es, mn_dist_info* info,
                               mn_error_detail* err) {
  switch (t) {
    case MN_TRI3: return dist_impl<MN_TRI3>(conn, M, base, N, comm, mem, ns, es, info, err);
    case MN_QUAD4: return dist_impl<MN_QUAD4>(conn, M, base, N, comm, mem, ns, es, info, err);
    case MN_TET4: return dist_impl<MN_TET4>(conn, M, base, N, comm, mem, ns, es, info, err);
    default: return dist_impl<MN_HEX8>(conn, M, base, N, comm, mem, ns, es, info, err);
  }
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

template <int T, int BINS>
static mn_status dist_p2p_impl(const int32_t* conn, int64_t M, int64_t base, int64_t N, mn_symm* h, Mem& mem,
                               mn_csr* node_slice, mn_csr* elem_slice, mn_dist_info* info, mn_error_detail* err) {
  constexpr int K = Elem<T>::K;
  cudaStream_t s = mem.s;
  const mn_comm* comm = &h->comm;
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
  int64_t nnz2[2] = {0, 0};
  uint64_t ew = ERR_NONE;
  int64_t in = 0, own = 0, own0 = 0;
  size_t pairs_bytes = 0;
  int32_t* relems = nullptr;
  // staging: all-gather rows + per-destination pointer tables; workspace: err, tickets, histogram,
  // bases, look-back status words
  int64_t* dx = (int64_t*)mem.get((size_t)W * (G + 1) * 8 + (size_t)G * 16);
  if (!dx) return MN_ERR_OOM;
  void** dptr = (void**)(dx + (size_t)W * (G + 1));
  const int64_t tiles = tiles_of(Pe, kTile);
  Arena ar;
  unsigned long long* errw = ar.take<unsigned long long>(2);
  uint32_t* tickets = ar.take<uint32_t>(8);
  unsigned long long* hist = ar.take<unsigned long long>(BINS);
  uint64_t* bases = ar.take<uint64_t>(BINS);
  uint64_t* status = ar.take<uint64_t>((size_t)(tiles ? tiles : 1) * BINS);
  const size_t head = ar.off;
  char* ws = (char*)mem.get(ar.off);
  if (!ws) local = MN_ERR_OOM;
  if (local == MN_OK) {
    errw = (unsigned long long*)(ws + (size_t)errw); tickets = (uint32_t*)(ws + (size_t)tickets);
    hist = (unsigned long long*)(ws + (size_t)hist); bases = (uint64_t*)(ws + (size_t)bases);
    status = (uint64_t*)(ws + (size_t)status);
    // ---- 1. validation + incidence counts per owner (one read of conn) ----
    if (cudaMemsetAsync(ws, 0, head, s) != cudaSuccess || cudaMemsetAsync(errw, 0xFF, 8, s) != cudaSuccess)
      local = MN_ERR_CUDA;
    if (local == MN_OK && M > 0) {
      if (launch("hist_validate", 4.0 * P.K * M, s, [&] {
            k_hist_validate<T, BINS, false><<<hist_grid(M), 256, 0, s>>>(conn, M, N, base, P.dp, 1, chunk, hist, errw);
          }) != cudaSuccess)
        local = MN_ERR_CUDA;
    }
    if (local == MN_OK &&
        (cudaMemcpyAsync(hh.data(), hist, BINS * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
         cudaMemcpyAsync(host, errw, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
         cudaStreamSynchronize(s) != cudaSuccess))
      local = MN_ERR_CUDA;
    if (local == MN_OK) ew = host[0];
  }
  // ---- 2. count exchange + plan (the lowest error over all ranks is returned by every rank) ----
  row[0] = (int64_t)ew;
  row[1] = local;
  if (local == MN_OK && ew == ERR_NONE)
    for (int g = 0; g < G; ++g) row[2 + g] = (int64_t)hh[g];
  MN_CUDA(cudaMemcpyAsync(dx, row.data(), (size_t)W * 8, cudaMemcpyHostToDevice, s));
  if (comm->allgather(comm->ctx, dx, dx + W, (size_t)W * 8, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  MN_CUDA(cudaMemcpyAsync(all.data(), dx + W, (size_t)W * G * 8, cudaMemcpyDeviceToHost, s));
  MN_CUDA(cudaStreamSynchronize(s));
  st = dist_plan(G, self, all.data(), rc.data(), rr.data(), err);
  if (st != MN_OK) goto done;
  // ---- 3. receive layouts of every rank (all ranks compute all of them), heap capacity ----
  {
    auto cnt = [&](int r, int g) { return all[(size_t)r * W + 2 + g]; };
    auto pbytes = [](int64_t n) { return ((size_t)n * 8 + 255) & ~(size_t)255; };   // pairs region
    size_t need = 0;
    std::vector<int64_t> offp(G, 0), offr(G, 0), ing(G, 0);
    for (int g = 0; g < G; ++g) {
      for (int r = 0; r < G; ++r) ing[g] += cnt(r, g);
      need = std::max(need, pbytes(ing[g]) + (size_t)(ing[g] - cnt(g, g)) * 4 * K + 256);
      // where this rank's bucket for g starts in g's pairs region, and in g's row table (rows are
      // kept for remote sources only: sources after g skip g's own block)
      for (int r = 0; r < self; ++r) offp[g] += cnt(r, g);
      offr[g] = offp[g] - (self > g ? cnt(g, g) : 0);
    }
    in = ing[self];
    own = cnt(self, self);
    own0 = offp[self];
    pairs_bytes = pbytes(in);
    st = symm_reserve(h, need, s);
    if (st != MN_OK) goto done;
    for (int g = 0; g < G; ++g) {
      dsth[g] = reinterpret_cast<uint64_t*>(h->peer[g]) + offp[g];
      rowh[g] = g == self ? nullptr : reinterpret_cast<int32_t*>(h->peer[g] + pbytes(ing[g])) + offr[g] * K;
    }
  }
  // ---- 4. fused bucket-and-send: one onesweep pass storing into the owners' heaps ----
  MN_CUDA(cudaMemcpyAsync(dptr, dsth.data(), (size_t)G * 8, cudaMemcpyHostToDevice, s));
  MN_CUDA(cudaMemcpyAsync(dptr + G, rowh.data(), (size_t)G * 8, cudaMemcpyHostToDevice, s));
  if (M > 0) {
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
    MN_CUDA(launch("bucket_send_p2p", 4.0 * Pe + 8.0 * Pe, s, [&] {
      kern<<<(unsigned)tiles, kPassThreads, smem, s>>>(pe);
    }));
  }
  // ---- 5. barrier: every rank's stores into this heap are complete past this all-gather ----
  MN_CUDA(cudaMemcpyAsync(dx, nnz2, 8, cudaMemcpyHostToDevice, s));
  if (comm->allgather(comm->ctx, dx, dx + 2, 8, (mn_stream)s) != 0) { st = MN_ERR_COMM; goto done; }
  // ---- 6. local finish over the heap (pairs in source-rank order, remote rows + their ids) ----
  {
    const int64_t nr = in - own;
    const uint64_t* hp = (const uint64_t*)h->local;
    const int32_t* hr = (const int32_t*)(h->local + pairs_bytes);
    if (nr > 0) {
      relems = (int32_t*)mem.get((size_t)nr * 4);
      if (!relems) { st = MN_ERR_OOM; goto done; }
      MN_CUDA(launch("remote_elems", 12.0 * nr, s, [&] {
        k_remote_elems<<<stream_grid(nr), 256, 0, s>>>(hp, nr, own0, own, relems);
      }));
    }
    if (in > INT32_MAX) { st = MN_ERR_CAPACITY; goto done; }
    st = dist_finish_impl<T>(pair_src(hp, in), in, relems, hr, nr, conn, base, M, N, lo, hi, mem, node_slice,
                             elem_slice);
    if (st != MN_OK) goto done;
    mem.put(relems);
    relems = nullptr;
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
  }
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
  mem.put(relems);
  mn_csr_release(node_slice, (mn_stream)s);
  mn_csr_release(elem_slice, (mn_stream)s);
  return st;
}

static mn_status dist_p2p_dispatch(mn_elem_type t, const int32_t* conn, int64_t M, int64_t base, int64_t N, mn_symm* h,
                                   Mem& mem, mn_csr* ns, mn_csr* es, mn_dist_info* info, mn_error_detail* err) {
  const bool b512 = h->comm.world > 256;
#define MN_P2P(TT) \
  return b512 ? dist_p2p_impl<TT, 512>(conn, M, base, N, h, mem, ns, es, info, err) \
              : dist_p2p_impl<TT, 256>(conn, M, base, N, h, mem, ns, es, info, err)
  switch (t) {
    case MN_TRI3: MN_P2P(MN_TRI3);
    case MN_QUAD4: MN_P2P(MN_QUAD4);
    case MN_TET4: MN_P2P(MN_TET4);
    default: MN_P2P(MN_HEX8);
  }
#undef MN_P2P
}
