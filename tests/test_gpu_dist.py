"""GPU tests of the multi-GPU building blocks (mn_dist_bucket / mn_dist_finish) on one B200:
G "virtual ranks" run one after another on the same device, the all-to-all replaced by slicing
and concatenating in source-rank order; the concatenated slices must equal the oracle CSR bit for
bit.  Plus the real torch.distributed NCCL path at world size 1."""
import os
import socket

import numpy as np
import pytest
import torch

import meshgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1604_04689_b200 import build
    build.build()


def _virtual_ranks(conn, et, N, G):
    import paper_1604_04689_b200 as mn
    from paper_1604_04689_b200.dist import owner_range
    M = conn.shape[0]
    sent, shards = [], []
    for r in range(G):
        s0, s1 = r * M // G, (r + 1) * M // G
        shard = conn[s0:s1].contiguous()
        pairs, cnt, relems, rows, rcnt = mn.dist_bucket(shard, et, s0, N, G, r)
        assert rcnt[r] == 0
        sent.append((list(torch.split(pairs, cnt)), list(torch.split(relems, rcnt)), list(torch.split(rows, rcnt))))
        shards.append((shard, s0))
    node_parts, elem_parts = [], []
    node_base = elem_base = 0
    for g in range(G):
        lo, hi = owner_range(N, G, g)
        pin = torch.cat([sent[r][0][g] for r in range(G)])
        ein = torch.cat([sent[r][1][g] for r in range(G)])
        rin = torch.cat([sent[r][2][g] for r in range(G)])
        if pin.numel():
            own = pin >> 32        # bucket g must hold exactly the incidences owned by rank g
            assert bool(((own >= lo) & (own < hi)).all())
        if ein.numel() > 1:
            assert bool((ein[1:] > ein[:-1]).all())   # remote rows: element ids ascending
        (no, ni), (eo, ei) = mn.dist_finish(et, pin, ein, rin, shards[g][0], shards[g][1], N, lo, hi)
        node_parts.append((no[:-1] + node_base, ni))
        elem_parts.append((eo[:-1] + elem_base, ei))
        node_base += ni.numel()
        elem_base += ei.numel()
    no = torch.cat([p[0] for p in node_parts] + [torch.tensor([node_base], device="cuda")])
    ni = torch.cat([p[1] for p in node_parts])
    eo = torch.cat([p[0] for p in elem_parts] + [torch.tensor([elem_base], device="cuda")])
    ei = torch.cat([p[1] for p in elem_parts])
    return (no, ni), (eo, ei)


@pytest.fixture(params=["radix", "transpose"])
def elem_path(request):
    import paper_1604_04689_b200 as mn
    mn.set_elem_path(request.param)
    yield request.param
    mn.set_elem_path("auto")


@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("name,et,make", [
    ("kuhn_9", meshgen.TET4, lambda: meshgen.kuhn_tets(9)),
    ("hex_9_perm", meshgen.HEX8, lambda: (meshgen.relabel(*meshgen.hex_grid(9), 5, 6), 1000)),
    ("sphere", meshgen.TRI3, lambda: meshgen.uv_sphere(64, 33)),
    ("quad", meshgen.QUAD4, lambda: meshgen.quad_grid(40, 50)),
])
def test_virtual_ranks_match_oracle(G, name, et, make, elem_path):
    conn, N = make()
    (no, ni), (eo, ei) = _virtual_ranks(conn.cuda(), et, N, G)
    ro, ri = oracle.node_csr(et, conn, N)
    so, si = oracle.elem_csr(et, conn, N)
    assert np.array_equal(no.cpu().numpy(), ro) and np.array_equal(ni.cpu().numpy(), ri)
    assert np.array_equal(eo.cpu().numpy(), so) and np.array_equal(ei.cpu().numpy(), si)


@pytest.mark.parametrize("cap", [32, 96])
@pytest.mark.parametrize("G", [2, 3])
def test_virtual_ranks_chunk_bucket_fallback(G, cap):
    """The finish's chunk-bucketed transpose with small fixed capacities: overflowing buckets take
    the guarded counted path; the slices still concatenate to the oracle's CSRs."""
    import paper_1604_04689_b200 as mn
    conn, N = meshgen.kuhn_tets(12)
    mn.set_elem_path("transpose")
    mn.set_chunk_cap(cap)
    try:
        (no, ni), (eo, ei) = _virtual_ranks(conn.cuda(), meshgen.TET4, N, G)
    finally:
        mn.set_chunk_cap(0)
        mn.set_elem_path("auto")
    ro, ri = oracle.node_csr(meshgen.TET4, conn, N)
    so, si = oracle.elem_csr(meshgen.TET4, conn, N)
    assert np.array_equal(no.cpu().numpy(), ro) and np.array_equal(ni.cpu().numpy(), ri)
    assert np.array_equal(eo.cpu().numpy(), so) and np.array_equal(ei.cpu().numpy(), si)


def test_virtual_ranks_config5_shape_small(elem_path):
    """Config 5's recipe (Kuhn, natural order) at 40^3, 8 ranks: equals the 1-GPU CSR."""
    import paper_1604_04689_b200 as mn
    conn, N = meshgen.kuhn_tets(40, device="cuda")
    ref = mn.find_neighbors(conn, "tet4", N)
    got = _virtual_ranks(conn, meshgen.TET4, N, 8)
    for a, b in zip(ref, got):
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.slow
def test_virtual_ranks_full_config5():
    """Full config 5 (Kuhn 320^3, 196.6 M tets) as 8 virtual ranks on one GPU, through the stage
    entry points: the concatenated slices equal the 1-GPU CSRs bit for bit."""
    import paper_1604_04689_b200 as mn
    et, conn, N = meshgen.make_config(5, device="cuda")
    ref = mn.find_neighbors(conn, et, N)
    ref = [(a.cpu(), b.cpu()) for a, b in ref]
    torch.cuda.empty_cache()
    got = _virtual_ranks(conn, et, N, 8)
    for a, b in zip(ref, got):
        assert torch.equal(a[0], b[0].cpu()) and torch.equal(a[1], b[1].cpu())


def test_bucket_reports_invalid_with_global_ids():
    import paper_1604_04689_b200 as mn
    conn = torch.tensor([[0, 1, 2], [1, 2, 9]], dtype=torch.int32).cuda()
    with pytest.raises(mn.MeshError) as ei:
        mn.dist_bucket(conn, "tri3", 1000, 5, 2, 0)
    assert (ei.value.code, ei.value.elem, ei.value.pos) == (2, 1001, 2)


def test_nccl_world_size_one():
    import torch.distributed as dist

    import paper_1604_04689_b200 as mn
    from paper_1604_04689_b200.dist import find_neighbors_dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        conn, N = meshgen.kuhn_tets(12, device="cuda")
        from paper_1604_04689_b200.dist import comm_for, release_comms
        res = find_neighbors_dist(conn, "tet4", 0, N)
        ref = mn.find_neighbors(conn, "tet4", N)
        assert (res.lo, res.hi) == (0, N)
        assert torch.equal(res.node[0], ref[0][0]) and torch.equal(res.node[1], ref[0][1])
        assert torch.equal(res.elem[0], ref[1][0]) and torch.equal(res.elem[1], ref[1][1])
        assert res.sent_bytes == 0 and res.own_incidences == 4 * conn.shape[0]
        assert (res.node_nnz_total, res.elem_nnz_total) == (ref[0][1].numel(), ref[1][1].numel())
        # SURVEY §8(b)'s single-output forms over the raw ncclComm_t
        h = comm_for().handle
        (o, i), lo, hi, gb = mn.find_neighbors_dist_nccl(conn, "tet4", 0, N, h, "node")
        assert (lo, hi, gb) == (0, N, 0) and torch.equal(o, ref[0][0]) and torch.equal(i, ref[0][1])
        (o, i), lo, hi, gb = mn.find_neighbors_dist_nccl(conn, "tet4", 0, N, h, "elem")
        assert (lo, hi, gb) == (0, N, 0) and torch.equal(o, ref[1][0]) and torch.equal(i, ref[1][1])
        # a validation error comes back through the exchange's error reduction
        bad = conn.clone()
        bad[77, 2] = N + 3
        for p2p in (False, True):
            with pytest.raises(mn.MeshError) as ei:
                find_neighbors_dist(bad, "tet4", 0, N, p2p=p2p)
            assert (ei.value.code, ei.value.elem, ei.value.pos) == (mn.MN_ERR_INDEX_OUT_OF_RANGE, 77, 2)
        # the fused bucket-and-send path over the symmetric heap (world 1: the own heap only)
        for _ in range(2):
            res = find_neighbors_dist(conn, "tet4", 0, N, p2p=True)
            assert torch.equal(res.node[0], ref[0][0]) and torch.equal(res.node[1], ref[0][1])
            assert torch.equal(res.elem[0], ref[1][0]) and torch.equal(res.elem[1], ref[1][1])
        release_comms()
    finally:
        dist.destroy_process_group()


def _spawn_worker(rank, world, port, q, p2p=False):
    import torch.distributed as dist

    import paper_1604_04689_b200 as mn
    from paper_1604_04689_b200.dist import find_neighbors_dist, gather_global
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ok = True
        for et, (conn, N) in ((meshgen.HEX8, (meshgen.relabel(*meshgen.hex_grid(14), 21, 22), 15 ** 3)),
                              (meshgen.TET4, meshgen.kuhn_tets(11))):
            M = conn.shape[0]
            s0, s1 = rank * M // world, (rank + 1) * M // world
            res = find_neighbors_dist(conn[s0:s1].contiguous().cuda(), et, s0, N, p2p=p2p)
            (no, ni), (eo, ei) = gather_global(res, N)
            ro, ri = oracle.node_csr(et, conn, N)
            so, si = oracle.elem_csr(et, conn, N)
            ok &= (np.array_equal(no.cpu().numpy(), ro) and np.array_equal(ni.cpu().numpy(), ri)
                   and np.array_equal(eo.cpu().numpy(), so) and np.array_equal(ei.cpu().numpy(), si))
            ok &= res.node_nnz_total == len(ri) and res.elem_nnz_total == len(si)
        # an invalid element in the last shard: every rank raises the same (global) error
        conn, N = meshgen.kuhn_tets(6)
        M = conn.shape[0]
        bad = conn.clone()
        bad[M - 5, 1] = bad[M - 5, 0]
        if world == 3:                 # a lower error in the middle shard
            bad[M // 2, 3] = -4
        s0, s1 = rank * M // world, (rank + 1) * M // world
        try:
            find_neighbors_dist(bad[s0:s1].contiguous().cuda(), "tet4", s0, N, p2p=p2p)
            ok = False
        except mn.MeshError as e:
            exp = (mn.MN_ERR_INDEX_OUT_OF_RANGE, M // 2, 3) if world == 3 else (mn.MN_ERR_DEGENERATE, M - 5, 1)
            ok &= (e.code, e.elem, e.pos) == exp
        from paper_1604_04689_b200.dist import release_comms
        release_comms()
        q.put((rank, bool(ok), res.sent_bytes))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_real_kernels_multi_rank_one_gpu(world, p2p):
    """The product dist path (mn_find_neighbors_dist through the C ABI) with `world` ranks sharing
    cuda:0; the exchange callbacks are host-staged over gloo (NCCL needs one GPU per rank); the
    globally lowest validation error is raised on every rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_spawn_worker, args=(r, world, port, q, p2p)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in out:
        assert ok, f"rank {rank}: {info}"


def test_bench_multi_rank_path_one_gpu():
    """bench.py's N>1 code path (sharded config 3, dist exchange, max-over-ranks timing, JSON line)
    with 2 ranks on one GPU over gloo."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MN_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0 and line["roofline"]["achieved"] > 0


def _edge_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1604_04689_b200 as mn
    from paper_1604_04689_b200.dist import find_neighbors_dist, gather_global, release_comms
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ok = True
        cases = [
            ("two tets, empty shards", meshgen.TET4, (torch.tensor([[0, 1, 2, 3], [1, 2, 3, 4]], dtype=torch.int32), 5)),
            ("N < world", meshgen.TRI3, (torch.tensor([[0, 1, 2]], dtype=torch.int32), 3)),
            ("isolated tail nodes", meshgen.QUAD4, (meshgen.quad_grid(3, 4)[0], 40)),
            ("empty mesh", meshgen.HEX8, (torch.zeros((0, 8), dtype=torch.int32), 11)),
            ("fan hub owned by rank 0", meshgen.TRI3, meshgen.nonmanifold_fan(300)),
        ]
        cases.append(("kuhn 9 (coherent)", meshgen.TET4, meshgen.kuhn_tets(9)))
        cases.append(("hex 6 relabelled", meshgen.HEX8, (meshgen.relabel(*meshgen.hex_grid(6), 3, 4), 343)))
        for (name, et, (conn, N)), path in [(c, p) for c in cases for p in ("auto", "radix", "transpose")]:
            mn.set_elem_path(path)   # radix: every shard "without locality"; transpose: "with"
            M = conn.shape[0]
            s0, s1 = rank * M // world, (rank + 1) * M // world
            ro, ri = oracle.node_csr(et, conn, N)
            so, si = oracle.elem_csr(et, conn, N)
            for p2p in (False, True):
                res = find_neighbors_dist(conn[s0:s1].contiguous().cuda(), et, s0, N, p2p=p2p)
                (no, ni), (eo, ei) = gather_global(res, N)
                good = (np.array_equal(no.cpu().numpy(), ro) and np.array_equal(ni.cpu().numpy(), ri)
                        and np.array_equal(eo.cpu().numpy(), so) and np.array_equal(ei.cpu().numpy(), si))
                if not good:
                    q.put((rank, False, f"{name} {path} p2p={p2p}"))
                    ok = False
        mn.set_elem_path("auto")
        release_comms()
        q.put((rank, bool(ok), "edge cases"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_dist_edge_cases_multi_rank_one_gpu():
    """Both exchange modes through the C ABI with 3 ranks on one GPU: shards without elements,
    fewer nodes than ranks, nodes used by no element, an empty mesh, a 300-valent hub."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_edge_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in out:
        assert ok, f"rank {rank}: {info}"


# ------------------------------------------------------------------------------------------------
# The PRODUCT multi-GPU path (mn_find_neighbors_dist) with G ranks as G threads of one process on
# one GPU: a thread-based mn_comm (host-staged all-gather / all-to-all(v), threading barriers)
# stands in for NCCL, each rank on its own CUDA stream.
# ------------------------------------------------------------------------------------------------
class _ThreadComm:
    def __init__(self, shared, rank):
        import paper_1604_04689_b200 as mn
        self.sh, self.rank = shared, rank
        self.struct = mn.Comm()
        self.struct.rank, self.struct.world = rank, shared["world"]
        self._ag = mn.ALLGATHER_FN(self._allgather)
        self._a2a = mn.ALLTOALLV_FN(self._alltoallv)
        self.struct.allgather, self.struct.alltoallv = self._ag, self._a2a

    def _allgather(self, ctx, d_send, d_recv, nbytes, stream):
        import paper_1604_04689_b200 as mn
        try:
            sh, W = self.sh, self.sh["world"]
            h = torch.empty(nbytes, dtype=torch.uint8)
            mn.memcpy_sync(h.data_ptr(), d_send, nbytes, stream)
            sh["parts"][self.rank] = h
            sh["bar"].wait()
            cat = torch.cat([sh["parts"][g] for g in range(W)])
            mn.memcpy_sync(d_recv, cat.data_ptr(), nbytes * W, stream)
            sh["bar"].wait()
            return 0
        except Exception:  # noqa: BLE001
            sh["bar"].abort()
            return 1

    def _alltoallv(self, ctx, ops, n_ops, stream):
        import paper_1604_04689_b200 as mn
        try:
            sh, W = self.sh, self.sh["world"]
            for o in range(n_ops):
                op = ops[o]
                eb = int(op.elem_bytes)
                for g in range(W):
                    n = int(op.send_counts[g]) * eb
                    h = torch.empty(n, dtype=torch.uint8)
                    if n:
                        mn.memcpy_sync(h.data_ptr(), op.send + int(op.send_displs[g]) * eb, n, stream)
                    sh["box"][(self.rank, g, o)] = h
                sh["bar"].wait()
                for g in range(W):
                    h = sh["box"][(g, self.rank, o)]
                    n = int(op.recv_counts[g]) * eb
                    assert h.numel() == n
                    if n:
                        mn.memcpy_sync(op.recv + int(op.recv_displs[g]) * eb, h.data_ptr(), n, stream)
                sh["bar"].wait()
            return 0
        except Exception:  # noqa: BLE001
            sh["bar"].abort()
            return 1


def _threaded_ranks(conn, et, N, G):
    import threading

    import paper_1604_04689_b200 as mn
    M = conn.shape[0]
    shared = {"world": G, "parts": [None] * G, "box": {}, "bar": threading.Barrier(G)}
    results, errors = [None] * G, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            comm = _ThreadComm(shared, r)
            s0, s1 = r * M // G, (r + 1) * M // G
            with torch.cuda.stream(s):
                shard = conn[s0:s1].contiguous()
                results[r] = mn.find_neighbors_dist_comm(shard, et, s0, N, comm.struct, stream=s)
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append((r, repr(e)))
            shared["bar"].abort()

    torch.cuda.synchronize()   # conn is complete before the ranks' streams read it
    threads = [threading.Thread(target=run, args=(r,)) for r in range(G)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    out = []
    for which in (0, 1):
        offs, idxs, tot = [], [], 0
        for r in range(G):
            off, idx = results[r][which]
            offs.append(off[:-1] + tot)
            idxs.append(idx)
            tot += idx.numel()
        out.append((torch.cat(offs + [torch.tensor([tot], device=offs[0].device)]), torch.cat(idxs)))
    return out, [results[r][2] for r in range(G)]


@pytest.mark.parametrize("G", [2, 3, 5])
@pytest.mark.parametrize("name,et,make", [
    ("kuhn_10", meshgen.TET4, lambda: meshgen.kuhn_tets(10)),
    ("hex_8_perm", meshgen.HEX8, lambda: (meshgen.relabel(*meshgen.hex_grid(8), 5, 6), 729)),
])
def test_product_path_threaded_ranks(G, name, et, make):
    conn, N = make()
    (no, ni), (eo, ei) = _threaded_ranks(conn.cuda(), et, N, G)[0]
    ro, ri = oracle.node_csr(et, conn, N)
    so, si = oracle.elem_csr(et, conn, N)
    assert np.array_equal(no.cpu().numpy(), ro) and np.array_equal(ni.cpu().numpy(), ri)
    assert np.array_equal(eo.cpu().numpy(), so) and np.array_equal(ei.cpu().numpy(), si)


@pytest.mark.slow
def test_product_path_full_config5_eight_ranks():
    """Full config 5 through mn_find_neighbors_dist with 8 ranks (threads on one GPU): the
    concatenated slices equal the 1-GPU CSRs bit for bit; remote traffic is the boundary layer."""
    import paper_1604_04689_b200 as mn
    et, conn, N = meshgen.make_config(5, device="cuda")
    ref = [(a.cpu(), b.cpu()) for a, b in mn.find_neighbors(conn, et, N)]
    torch.cuda.empty_cache()
    got, infos = _threaded_ranks(conn, et, N, 8)
    for a, b in zip(ref, got):
        assert torch.equal(a[0], b[0].cpu()) and torch.equal(a[1], b[1].cpu())
    own = sum(i.own_incidences for i in infos)
    assert 0.95 < own / (4 * conn.shape[0]) < 1.0
