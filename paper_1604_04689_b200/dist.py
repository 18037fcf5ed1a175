"""Multi-GPU one-ring neighbours: one process per GPU, elements sharded.

Each rank holds a contiguous element shard (global element base given).  Nodes are owned in
contiguous ranges [r*ceil(N/G), (r+1)*ceil(N/G)).  Per call:

  1. mn_dist_bucket   (CUDA)  validate the shard, create its (node, element) incidences and
                              stably bucket them by owner rank (one onesweep pass, pairs created
                              from conn); one row per (remote destination, element) goes along;
  2. count exchange           all_to_all of the G (incidence, row) counts (NCCL over NVLink);
  3. payload exchange         all_to_all(v) of the pairs, the remote element ids and their rows,
                              received in source-rank order, so element ids stay ascending;
  4. mn_dist_finish   (CUDA)  element CSR slice by a stable sort on the local node id; node CSR
                              slice by the same per-node expansion + dedupe as the 1-GPU path, rows
                              read from the own shard (local elements) or the received table.

Only incidences travel (8 bytes each, plus 4(k+1) bytes per remote element row), never the 2E node
pairs per element; with a spatially coherent numbering almost everything stays on its rank.
The result on rank r is the CSR of nodes [lo_r, hi_r) with local offsets; concatenating the slices
in rank order (offsets shifted by the preceding ranks' nnz, returned as ``*_base``) is
bit-identical to the single-GPU CSR.

``ops`` is the per-rank compute: the CUDA library by default.  The exchange logic is independent
of it, which is what lets tests/test_dist_gloo.py drive this exact orchestration over the gloo
backend on CPU with a test-side stand-in for the two CUDA calls.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class DistResult:
    lo: int
    hi: int
    node: tuple          # (offsets int64[hi-lo+1], indices int32[nnz]) — local offsets
    elem: tuple
    node_base: int       # global offset of this slice in the single-GPU node CSR
    elem_base: int
    sent_pairs: int      # incidences this rank sent to other ranks (exchange volume)


def owner_range(num_nodes: int, world: int, rank: int):
    chunk = max(1, -(-num_nodes // world))
    lo = min(num_nodes, rank * chunk)
    hi = min(num_nodes, (rank + 1) * chunk)
    return lo, hi


class CudaOps:
    """The product compute: libmeshnbr's two dist entry points."""

    @staticmethod
    def bucket(conn_shard, etype, elem_base, num_nodes, world, rank):
        from . import dist_bucket
        return dist_bucket(conn_shard, etype, elem_base, num_nodes, world, rank)

    @staticmethod
    def finish(etype, pairs, row_elems, rows, conn_shard, elem_base, num_nodes, lo, hi):
        from . import dist_finish
        return dist_finish(etype, pairs, row_elems, rows, conn_shard, elem_base, num_nodes, lo, hi)


def _a2a(out, inp, out_splits, in_splits, group):
    """all_to_all_single; with a gloo group and CUDA tensors the exchange is staged through host
    memory (gloo has no CUDA all-to-all) — used to exercise the multi-rank path on one GPU."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        host_out = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(host_out, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(host_out)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)


def _all_gather(outs, inp, group):
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        host = [torch.empty(o.shape, dtype=o.dtype) for o in outs]
        dist.all_gather(host, inp.cpu(), group=group)
        for o, h in zip(outs, host):
            o.copy_(h)
    else:
        dist.all_gather(outs, inp, group=group)


def find_neighbors_dist(conn_shard: torch.Tensor, etype, global_elem_base: int, num_nodes: int,
                        group=None, ops=None) -> DistResult:
    ops = ops or CudaOps
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = conn_shard.device
    pairs, count, relems, rows, rcount = ops.bucket(conn_shard, etype, int(global_elem_base), int(num_nodes),
                                                   world, rank)
    k = rows.shape[1] if rows.dim() == 2 else 1
    # ---- count exchange: row g of `send` goes to rank g ----
    send = torch.tensor([[count[g], rcount[g]] for g in range(world)], dtype=torch.int64, device=dev)
    recv = torch.empty_like(send)
    _a2a(recv.view(-1), send.reshape(-1), None, None, group)
    recv = recv.reshape(world, 2).cpu()
    rc, rr = recv[:, 0].tolist(), recv[:, 1].tolist()
    # ---- payload exchange, received in source-rank order ----
    pairs_in = torch.empty(sum(rc), dtype=torch.int64, device=dev)
    relems_in = torch.empty(sum(rr), dtype=torch.int32, device=dev)
    rows_in = torch.empty((sum(rr), k), dtype=torch.int32, device=dev)
    _a2a(pairs_in, pairs, rc, list(count), group)
    _a2a(relems_in, relems, rr, list(rcount), group)
    _a2a(rows_in, rows, rr, list(rcount), group)
    del pairs, relems, rows
    lo, hi = owner_range(num_nodes, world, rank)
    node, elem = ops.finish(etype, pairs_in, relems_in, rows_in, conn_shard, int(global_elem_base),
                            num_nodes, lo, hi)
    # ---- global bases of the slices (exclusive scan of the per-rank nnz) ----
    mine = torch.tensor([node[1].numel(), elem[1].numel()], dtype=torch.int64, device=dev)
    allv = [torch.empty_like(mine) for _ in range(world)]
    _all_gather(allv, mine, group)
    allv = torch.stack(allv).cpu()
    node_base = int(allv[:rank, 0].sum())
    elem_base = int(allv[:rank, 1].sum())
    sent = sum(int(count[g]) for g in range(world) if g != rank)   # remote incidences
    return DistResult(lo, hi, node, elem, node_base, elem_base, sent)


def gather_global(res: DistResult, num_nodes: int, group=None):
    """Assemble the global CSRs on every rank (verification helper; moves everything)."""
    world = dist.get_world_size(group)
    out = []
    for which, base in ((res.node, res.node_base), (res.elem, res.elem_base)):
        off, idx = which
        glob_off = off[:-1] + base
        sizes = torch.tensor([glob_off.numel(), idx.numel()], dtype=torch.int64, device=off.device)
        allsz = [torch.empty_like(sizes) for _ in range(world)]
        _all_gather(allsz, sizes, group)
        allsz = torch.stack(allsz).cpu()
        mo, mi = int(allsz[:, 0].max()), int(allsz[:, 1].max())
        po = torch.zeros(mo, dtype=torch.int64, device=off.device)
        po[: glob_off.numel()] = glob_off
        pi = torch.zeros(mi, dtype=torch.int32, device=off.device)
        pi[: idx.numel()] = idx
        offs = [torch.empty_like(po) for _ in range(world)]
        idxs = [torch.empty_like(pi) for _ in range(world)]
        _all_gather(offs, po, group)      # padded to equal sizes (gloo needs that)
        _all_gather(idxs, pi, group)
        offs = [o[: int(s[0])] for o, s in zip(offs, allsz)]
        idxs = [x[: int(s[1])] for x, s in zip(idxs, allsz)]
        total = int(allsz[:, 1].sum())
        full_off = torch.cat(offs + [torch.tensor([total], dtype=torch.int64, device=off.device)])
        out.append((full_off, torch.cat(idxs)))
    return out[0], out[1]
