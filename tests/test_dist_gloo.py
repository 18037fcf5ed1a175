"""Multi-process (world size 2 and 3, gloo, CPU) tests of the multi-GPU protocol of
mn_find_neighbors_dist (include/meshnbr.h).

* The host half of the library's step 2, mn_dist_plan (exported, host-only C++), runs on every rank
  over rows all-gathered with gloo: receive counts and the global error must agree with what is
  computed directly from the whole mesh, and every rank must return the same (lowest) error.
* A test-side model of the whole call (numpy stand-ins for the two per-rank CUDA steps, written
  from oracle/stages.py; the library's own plan for step 2; gloo for the exchanges, with the
  owner's bucket kept in place as the library does) must concatenate to the oracle's CSRs.
The CUDA path itself runs multi-rank in tests/test_gpu_dist.py (ranks sharing one GPU)."""
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

NONE = (1 << 64) - 1


def _owner(nodes, N, world):
    chunk = max(1, -(-N // world))
    return np.minimum(np.asarray(nodes, dtype=np.int64) // chunk, world - 1)


def _err_word(conn_shard, N, base):
    """Lowest (element << 5 | repeated << 4 | position) of the shard, or all ones (the encoding of
    include/meshnbr.h mn_dist_plan), from the oracle's validation (global element ids)."""
    code, e, p = oracle.validate(meshgen.TET4 if conn_shard.shape[1] == 4 else meshgen.TRI3, conn_shard, N)
    if code == oracle.OK:
        return NONE
    return ((e + base) << 5) | ((1 if code == oracle.ERR_DEGENERATE else 0) << 4) | p


def _row(conn_shard, N, world, rank, base):
    """This rank's step-2 row: [error word, status, incidences per owner, remote rows per owner]."""
    conn = np.asarray(conn_shard)
    ew = _err_word(conn, N, base)
    counts = np.zeros(world, np.int64)
    rows = np.zeros(world, np.int64)
    if ew == NONE and conn.size:
        own = _owner(conn.reshape(-1), N, world)
        counts = np.bincount(own, minlength=world).astype(np.int64)
        per_elem = own.reshape(conn.shape)
        for g in range(world):
            if g != rank:
                rows[g] = int((per_elem == g).any(1).sum())
    return np.concatenate([[np.int64(np.uint64(ew).view(np.int64))], [0], counts, rows]).astype(np.int64)


def _gather_rows(row, world):
    t = torch.from_numpy(row)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    return torch.stack(outs).numpy()


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ------------------------------------------------------------------------------------------------
# 1. mn_dist_plan over gloo
# ------------------------------------------------------------------------------------------------
def _plan_worker(rank, world, port, bad, q):
    _init(rank, world, port)
    try:
        import paper_1604_04689_b200 as mn
        conn, N = meshgen.kuhn_tets(4)
        conn = conn.numpy()
        for (e, p, v) in bad:                      # global (element, position, value) corruptions
            conn[e, p] = v if v >= 0 else conn[e, -v - 1]
        M = conn.shape[0]
        s0, s1 = rank * M // world, (rank + 1) * M // world
        allrows = _gather_rows(_row(conn[s0:s1], N, world, rank, s0), world)
        st, rc, rr, ee, ep = mn.dist_plan(world, rank, allrows)
        code, oe, opos = oracle.validate(meshgen.TET4, conn, N)
        if code == oracle.OK:
            own = _owner(conn.reshape(-1), N, world).reshape(conn.shape)
            exp_rc = [int((own[r * M // world:(r + 1) * M // world] == rank).sum()) for r in range(world)]
            exp_rr = [0 if r == rank else int((own[r * M // world:(r + 1) * M // world] == rank).any(1).sum())
                      for r in range(world)]
            ok = st == mn.MN_OK and rc == exp_rc and rr == exp_rr
        else:
            exp = {oracle.ERR_RANGE: mn.MN_ERR_INDEX_OUT_OF_RANGE, oracle.ERR_DEGENERATE: mn.MN_ERR_DEGENERATE}[code]
            ok = (st, ee, ep) == (exp, oe, opos)
        q.put((rank, bool(ok), (st, rc, rr, ee, ep)))
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


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("bad", [
    [],                                    # valid: receive counts and row counts
    [(300, 2, 10 ** 6)],                   # out of range in the last shard only
    [(350, 1, -1), (20, 3, 125)],          # degenerate late, range early: the early one wins everywhere
    [(100, 3, -2), (100, 1, 125)],         # same element: range (pos 1) before repeated node (pos 3)
])
def test_dist_plan_gloo(world, bad):
    """mn_dist_plan on every rank over gloo-gathered rows: per-source receive counts equal the
    incidences this rank owns in each shard; a validation error anywhere is reported identically
    (lowest global element, range before repeated node) by every rank."""
    for rank, ok, info in _spawn(_plan_worker, world, bad):
        assert ok, f"rank {rank}: {info}"


# ------------------------------------------------------------------------------------------------
# 2. model of the whole call: partition, in-place own bucket, exchange, finish, bases
# ------------------------------------------------------------------------------------------------
def _bucket_model(conn, etype, base, N, world, rank):
    """Stand-in for steps 1 and 3 (CUDA in the product): incidences (node << 32 | element) stably
    bucketed by owner, element-major inside a bucket; each REMOTE incidence travels with its
    element's row (the product's bucket-and-send); the own bucket stays in place."""
    k = stages.ARITY[etype]
    en, ee = stages.expand_elem_pairs(etype, conn)
    own = _owner(en, N, world)
    order = np.argsort(own, kind="stable")
    pairs = ((en.astype(np.int64) << 32) | (ee.astype(np.int64) + base))[order]
    owns, elems = own[order], ee[order]
    relems, rows = [], []
    for g in range(world):
        sel = elems[owns == g] if g != rank else np.zeros(0, np.int64)
        relems.append(sel + base)
        rows.append(conn.reshape(-1, k)[sel])
    return pairs, np.bincount(own, minlength=world), relems, rows


def _finish_model(etype, pairs, table, shard, base, lo, hi):
    """Stand-in for step 4: stable sort on the local node id (element CSR), per-node expansion +
    dedupe (node CSR), rows from the own shard or the received table."""
    nodes, elems = (pairs >> 32), (pairs & 0xFFFFFFFF)
    order = np.argsort(nodes - lo, kind="stable")
    nloc = hi - lo
    uk, cnt = stages.reduce_by_key_ones((nodes - lo)[order])
    eoff = stages.exclusive_scan(stages.dense_counts(uk, cnt, nloc))
    eidx = elems[order].astype(np.int32)
    adj = [set() for _ in range(nloc)]
    for a, e in zip(nodes.tolist(), elems.tolist()):
        row = shard[e - base].tolist() if 0 <= e - base < len(shard) else table[e]
        pa = row.index(a)
        for i, j in stages.EDGES[etype]:
            if i == pa:
                adj[a - lo].add(row[j])
            if j == pa:
                adj[a - lo].add(row[i])
    noff = stages.exclusive_scan([len(x) for x in adj])
    nidx = np.array([v for x in adj for v in sorted(x)], dtype=np.int32)
    return (noff, nidx), (eoff, eidx)


def _a2a_model(parts, world):
    """all_to_all(v) over gloo of per-destination numpy arrays (the own part is not sent)."""
    rank = dist.get_rank()
    send = [torch.from_numpy(np.ascontiguousarray(p)) if g != rank else torch.from_numpy(p[:0].copy())
            for g, p in enumerate(parts)]
    sizes = torch.tensor([s.numel() for s in send], dtype=torch.int64)
    allsz = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(allsz, sizes)
    rsz = [int(allsz[g][rank]) for g in range(world)]
    recv = torch.empty(sum(rsz), dtype=send[0].dtype)
    dist.all_to_all_single(recv, torch.cat(send), rsz, [s.numel() for s in send])
    return [r.numpy() for r in torch.split(recv, rsz)]


MESHES = {
    "kuhn5": (meshgen.TET4, lambda: meshgen.kuhn_tets(5)),
    "hexperm": (meshgen.HEX8, lambda: (meshgen.relabel(*meshgen.hex_grid(4), 9, 10), 125)),
    "sphere": (meshgen.TRI3, lambda: meshgen.uv_sphere(12, 7)),
}


def _model_worker(rank, world, port, name, q):
    _init(rank, world, port)
    try:
        import paper_1604_04689_b200 as mn
        et, make = MESHES[name]
        conn, N = make()
        conn = conn.numpy()
        k = stages.ARITY[et]
        M = conn.shape[0]
        s0, s1 = rank * M // world, (rank + 1) * M // world
        shard = conn[s0:s1]
        pairs, counts, relems, rows = _bucket_model(shard, et, s0, N, world, rank)
        row = np.concatenate([[-1, 0], counts, [len(r) for r in relems]]).astype(np.int64)   # aux: rows sent
        st, rc, rr, _, _ = mn.dist_plan(world, rank, _gather_rows(row, world))
        assert st == mn.MN_OK
        splits = np.split(pairs, np.cumsum(counts)[:-1])
        got = _a2a_model(splits, world)
        assert [len(x) for g, x in enumerate(got) if g != rank] == [c for g, c in enumerate(rc) if g != rank]
        got[rank] = splits[rank]                                 # own bucket read in place
        inp = np.concatenate(got)
        re = np.concatenate(_a2a_model([r.astype(np.int64) for r in relems], world))
        rw = np.concatenate(_a2a_model([r.reshape(-1).astype(np.int64) for r in rows], world)).reshape(-1, k)
        assert len(re) == sum(rr)
        from paper_1604_04689_b200.dist import owner_range
        lo, hi = owner_range(N, world, rank)
        (no, ni), (eo, ei) = _finish_model(et, inp, dict(zip(re.tolist(), rw.tolist())), shard, s0, lo, hi)
        nnz = torch.tensor([len(ni), len(ei)], dtype=torch.int64)
        alln = [torch.empty_like(nnz) for _ in range(world)]
        dist.all_gather(alln, nnz)
        nb = sum(int(x[0]) for x in alln[:rank])
        eb = sum(int(x[1]) for x in alln[:rank])
        ro, ri = oracle.node_csr(et, conn, N)
        so, si = oracle.elem_csr(et, conn, N)
        ok = (np.array_equal(no + nb, ro[lo:hi + 1]) and np.array_equal(ni, ri[ro[lo]:ro[hi]])
              and np.array_equal(eo + eb, so[lo:hi + 1]) and np.array_equal(ei, si[so[lo]:so[hi]]))
        q.put((rank, bool(ok), sum(int(c) for g, c in enumerate(counts) if g != rank)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(MESHES))
def test_dist_protocol_model_gloo(world, name):
    for rank, ok, info in _spawn(_model_worker, world, name):
        assert ok, f"rank {rank}: {info}"
        assert isinstance(info, int)
