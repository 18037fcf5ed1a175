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
