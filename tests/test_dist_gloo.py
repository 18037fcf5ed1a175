"""Multi-process (world size 2 and 3, gloo, CPU) test of the multi-GPU orchestration in
paper_1604_04689_b200/dist.py: owner ranges, count exchange, uneven all_to_all splits, source-rank
order of received pairs, slice bases.  The two per-rank compute calls (bucket / finish, CUDA in
the product) are replaced by a test-side numpy stand-in written from oracle/stages.py; the global
CSR assembled from the slices must equal the oracle's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import meshgen
import oracle
from oracle import stages


def _bits(N):
    b = 0
    x = max(N - 1, 0)
    while x:
        b += 1
        x >>= 1
    return max(b, 1)


class NumpyOps:
    """CPU stand-in with the C ABI's contract (include/meshnbr.h mn_dist_bucket / _finish)."""

    @staticmethod
    def bucket(conn_shard, etype, elem_base, N, world, rank):
        conn = conn_shard.numpy()
        k = stages.ARITY[etype]
        chunk = max(1, -(-N // world))
        en, ee = stages.expand_elem_pairs(etype, conn)          # element-major incidences
        own = np.minimum(en.astype(np.int64) // chunk, world - 1)
        order = np.argsort(own, kind="stable")
        pairs = ((en.astype(np.int64) << 32) | (ee.astype(np.int64) + elem_base))[order]
        owns, elems = own[order], ee[order]
        relems, rows, rcount = [], [], []
        for g in range(world):
            sel = np.unique(elems[owns == g]) if g != rank else np.zeros(0, dtype=np.int64)
            relems.append(sel + elem_base)
            rows.append(conn.reshape(-1, k)[sel])
            rcount.append(len(sel))
        return (torch.from_numpy(pairs.copy()), np.bincount(own, minlength=world).tolist(),
                torch.from_numpy(np.concatenate(relems).astype(np.int32)),
                torch.from_numpy(np.concatenate(rows).astype(np.int32).reshape(-1, k)), rcount)

    @staticmethod
    def finish(etype, pairs, relems, rows, conn_shard, elem_base, N, lo, hi):
        p = pairs.numpy()
        shard = conn_shard.numpy()
        table = {int(e): r for e, r in zip(relems.numpy().tolist(), rows.numpy().tolist())}
        nodes, elems = (p >> 32), (p & 0xFFFFFFFF)
        order = np.argsort(nodes - lo, kind="stable")
        nloc = hi - lo
        uk, cnt = stages.reduce_by_key_ones((nodes - lo)[order])
        eoff = stages.exclusive_scan(stages.dense_counts(uk, cnt, nloc))
        eidx = elems[order].astype(np.int32)
        adj = [set() for _ in range(nloc)]
        for a, e in zip(nodes.tolist(), elems.tolist()):
            row = shard[e - elem_base].tolist() if 0 <= e - elem_base < len(shard) else table[e]
            pa = row.index(a)
            for i, j in stages.EDGES[etype]:
                if i == pa:
                    adj[a - lo].add(row[j])
                if j == pa:
                    adj[a - lo].add(row[i])
        noff = stages.exclusive_scan([len(x) for x in adj])
        nidx = np.array([v for x in adj for v in sorted(x)], dtype=np.int32)
        return ((torch.from_numpy(noff), torch.from_numpy(nidx)),
                (torch.from_numpy(eoff), torch.from_numpy(eidx)))


MESHES = {
    "kuhn5": (meshgen.TET4, lambda: meshgen.kuhn_tets(5)),
    "hexperm": (meshgen.HEX8, lambda: (meshgen.relabel(*meshgen.hex_grid(4), 9, 10), 125)),
    "sphere": (meshgen.TRI3, lambda: meshgen.uv_sphere(12, 7)),
}


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_04689_b200.dist import find_neighbors_dist, gather_global, owner_range
        et, make = MESHES[name]
        conn, N = make()
        M = conn.shape[0]
        s0, s1 = rank * M // world, (rank + 1) * M // world
        res = find_neighbors_dist(conn[s0:s1].contiguous(), et, s0, N, ops=NumpyOps)
        assert (res.lo, res.hi) == owner_range(N, world, rank)
        (no, ni), (eo, ei) = gather_global(res, N)
        ok = True
        ro, ri = oracle.node_csr(et, conn, N)
        so, si = oracle.elem_csr(et, conn, N)
        ok &= np.array_equal(no.numpy(), ro) and np.array_equal(ni.numpy(), ri)
        ok &= np.array_equal(eo.numpy(), so) and np.array_equal(ei.numpy(), si)
        q.put((rank, bool(ok), res.sent_pairs))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(MESHES))
def test_dist_orchestration_gloo(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in out:
        assert ok, f"rank {rank}: {info}"
