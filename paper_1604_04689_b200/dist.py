"""Multi-GPU one-ring neighbours: one process per GPU, elements sharded.

The whole path runs inside the library call ``mn_find_neighbors_dist`` (include/meshnbr.h):
validate + bucket the shard's incidences by owner rank, one all-gather of the counts (and of the
validation words, so every rank returns the globally lowest error), one grouped all-to-all(v) of
the remote incidences, remote element ids and their rows, the local finish (element CSR slice by a
stable sort, node CSR slice by per-node expansion + dedupe), one all-gather of the slice nnz.

Nodes are owned in contiguous ranges [r*ceil(N/G), (r+1)*ceil(N/G)); an owner's own incidences are
read in place and never exchanged.  The result on rank r is the CSR of nodes [lo_r, hi_r) with
local offsets; concatenating the slices in rank order (offsets shifted by ``*_base``) is
bit-identical to the single-GPU CSR.

This module only supplies the library's exchange operations (an ``mn_comm``) for a torch process
group: over NCCL (the product path: the library drives its own NCCL communicator, bootstrapped by
broadcasting an ncclUniqueId over the group), or host-staged over gloo (several ranks sharing one
GPU in tests, where NCCL cannot run).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import (ALLGATHER_FN, ALLTOALLV_FN, Comm, _check, find_neighbors_dist_comm, find_neighbors_dist_p2p, load,
               memcpy_sync, symm_create, symm_destroy, symm_unmap)


@dataclass
class DistResult:
    lo: int
    hi: int
    node: tuple          # (offsets int64[hi-lo+1], indices int32[nnz]) — local offsets
    elem: tuple
    node_base: int       # global offset of this slice in the single-GPU node CSR
    elem_base: int
    sent_bytes: int      # payload bytes this rank sent to other ranks
    recv_bytes: int      # payload bytes it received
    own_incidences: int  # incidences it kept in place (not exchanged)
    node_nnz_total: int
    elem_nnz_total: int


def owner_range(num_nodes: int, world: int, rank: int):
    chunk = max(1, -(-num_nodes // world))
    lo = min(num_nodes, rank * chunk)
    hi = min(num_nodes, (rank + 1) * chunk)
    return lo, hi


class NcclComm:
    """The library's own NCCL communicator for a torch process group (NVLink / NVSwitch)."""

    def __init__(self, group=None):
        lib = load()
        if not lib.mn_nccl_available():
            raise RuntimeError("libnccl.so.2 could not be loaded by libmeshnbr")
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            _check(lib.mn_nccl_get_unique_id(ctypes.c_void_p(idt.data_ptr())))
        dev = torch.device("cuda", torch.cuda.current_device())
        buf = idt.to(dev) if dist.get_backend(group) == "nccl" else idt
        dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        idt = buf.cpu()
        self.handle = ctypes.c_void_p()
        _check(lib.mn_nccl_comm_init(ctypes.c_void_p(idt.data_ptr()), world, rank, ctypes.byref(self.handle)))
        self.struct = Comm()
        _check(lib.mn_comm_from_nccl(self.handle, ctypes.byref(self.struct)))

    def close(self):
        if self.handle:
            load().mn_nccl_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()


class HostComm:
    """Host-staged exchange over a gloo group: the callbacks copy the library's device buffers to
    host memory, run the gloo collective, and copy back (tests: several ranks sharing one GPU)."""

    def __init__(self, group=None):
        self.group = group
        self.struct = Comm()
        self.struct.rank = dist.get_rank(group)
        self.struct.world = dist.get_world_size(group)
        self._ag = ALLGATHER_FN(self._allgather)
        self._a2a = ALLTOALLV_FN(self._alltoallv)
        self.struct.allgather = self._ag
        self.struct.alltoallv = self._a2a

    def _allgather(self, ctx, d_send, d_recv, nbytes, stream):
        try:
            world = self.struct.world
            h = torch.empty(nbytes, dtype=torch.uint8)
            memcpy_sync(h.data_ptr(), d_send, nbytes, stream)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, h, group=self.group)
            cat = torch.cat(outs)
            memcpy_sync(d_recv, cat.data_ptr(), nbytes * world, stream)
            return 0
        except Exception:  # noqa: BLE001  (a failed exchange is MN_ERR_COMM in the library)
            return 1

    def _alltoallv(self, ctx, ops, n_ops, stream):
        try:
            world = self.struct.world
            for o in range(n_ops):
                op = ops[o]
                eb = int(op.elem_bytes)
                sc = [int(op.send_counts[g]) * eb for g in range(world)]
                rc = [int(op.recv_counts[g]) * eb for g in range(world)]
                send = torch.empty(sum(sc), dtype=torch.uint8)
                pos = 0
                for g in range(world):
                    if sc[g]:
                        memcpy_sync(send.data_ptr() + pos, op.send + int(op.send_displs[g]) * eb, sc[g], stream)
                    pos += sc[g]
                recv = torch.empty(sum(rc), dtype=torch.uint8)
                dist.all_to_all_single(recv, send, rc, sc, group=self.group)
                pos = 0
                for g in range(world):
                    if rc[g]:
                        memcpy_sync(op.recv + int(op.recv_displs[g]) * eb, recv.data_ptr() + pos, rc[g], stream)
                    pos += rc[g]
            return 0
        except Exception:  # noqa: BLE001
            return 1


_COMMS = {}


def comm_for(group=None):
    """The cached mn_comm provider of a process group: NCCL for an NCCL group, host-staged for gloo."""
    key = id(group) if group is not None else None
    if key not in _COMMS:
        _COMMS[key] = NcclComm(group) if dist.get_backend(group) == "nccl" else HostComm(group)
    return _COMMS[key]


_SYMMS = {}


def symm_for(group=None):
    """The cached symmetric receive heap of a process group (created collectively on first use)."""
    key = id(group) if group is not None else None
    if key not in _SYMMS:
        _SYMMS[key] = symm_create(comm_for(group).struct)
    return _SYMMS[key]


def release_comms():
    """Collective teardown: every rank unmaps the other heaps, a barrier, then frees its own."""
    for key, h in _SYMMS.items():
        symm_unmap(h)
    if _SYMMS:
        torch.cuda.synchronize()
        dist.barrier()
    for h in _SYMMS.values():
        symm_destroy(h)
    _SYMMS.clear()
    for c in _COMMS.values():
        if isinstance(c, NcclComm):
            c.close()
    _COMMS.clear()


def find_neighbors_dist(conn_shard: torch.Tensor, etype, global_elem_base: int, num_nodes: int,
                        group=None, stream=None, p2p: bool = False) -> DistResult:
    """This rank's CSR slices through the C ABI: mn_find_neighbors_dist (bucket, NCCL all-to-all,
    finish), or with p2p=True mn_find_neighbors_dist_p2p (the bucketing kernel stores straight into
    the owners' symmetric heaps over peer memory)."""
    comm = comm_for(group)
    if p2p:
        node, elem, info = find_neighbors_dist_p2p(conn_shard, etype, int(global_elem_base), int(num_nodes),
                                                   symm_for(group), stream)
    else:
        node, elem, info = find_neighbors_dist_comm(conn_shard, etype, int(global_elem_base), int(num_nodes),
                                                    comm.struct, stream)
    return DistResult(int(info.lo), int(info.hi), node, elem, int(info.node_base), int(info.elem_base),
                      int(info.sent_bytes), int(info.recv_bytes), int(info.own_incidences),
                      int(info.node_nnz_total), int(info.elem_nnz_total))


def _all_gather(outs, inp, group):
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        host = [torch.empty(o.shape, dtype=o.dtype) for o in outs]
        dist.all_gather(host, inp.cpu(), group=group)
        for o, h in zip(outs, host):
            o.copy_(h)
    else:
        dist.all_gather(outs, inp, group=group)


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


__all__ = ["DistResult", "owner_range", "NcclComm", "HostComm", "comm_for", "symm_for", "release_comms",
           "find_neighbors_dist", "gather_global"]
