"""GPU parity: every §8(a) row of the CUDA path (through the C ABI) against the oracle, element by
element, on seeded synthetic meshes; full-size configs on sampled vertices + properties that hold
at any size.  Bar: bit-exact (integer work)."""
import numpy as np
import pytest
import torch

import meshgen
import oracle
from oracle import stages

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1604_04689_b200 import build
    build.build()


def mn():
    import paper_1604_04689_b200 as m
    return m


def _perm_hex(n, node_seed, elem_seed):
    conn, N = meshgen.hex_grid(n)
    return meshgen.relabel(conn, N, node_seed, elem_seed), N


# Small/medium meshes: several onesweep tiles (4096 keys) and ragged tails, every element type.
SMALL = [
    ("tri_grid_32", meshgen.TRI3, lambda: meshgen.tri_grid(32, 32)),          # config 1
    ("tri_grid_77x41", meshgen.TRI3, lambda: meshgen.tri_grid(41, 77)),
    ("quad_grid_60x33", meshgen.QUAD4, lambda: meshgen.quad_grid(33, 60)),
    ("kuhn_11", meshgen.TET4, lambda: meshgen.kuhn_tets(11)),
    ("hex_13_perm", meshgen.HEX8, lambda: _perm_hex(13, 1604, 4689)),
    ("sphere_100x51", meshgen.TRI3, lambda: meshgen.uv_sphere(100, 51)),
    ("rand_tri", meshgen.TRI3, lambda: meshgen.random_mesh(meshgen.TRI3, 3000, 700, seed=5)),
    ("rand_tet_sparse", meshgen.TET4, lambda: meshgen.random_mesh(meshgen.TET4, 900, 5000, seed=6)),
    ("rand_hex", meshgen.HEX8, lambda: meshgen.random_mesh(meshgen.HEX8, 700, 3000, seed=8)),
    ("rand_quad_big_ids", meshgen.QUAD4, lambda: meshgen.random_mesh(meshgen.QUAD4, 800, 70000, seed=9)),
    ("fan5", meshgen.TRI3, lambda: meshgen.nonmanifold_fan(5)),
    ("single_tet", meshgen.TET4, lambda: (torch.tensor([[3, 1, 0, 2]], dtype=torch.int32), 4)),
    ("hex_big_ids", meshgen.HEX8, lambda: _perm_hex(9, 77, None)),
    # > 32 distinct neighbours with <= 256 raw entries: hash-set overflow -> block path
    ("rand_tet_dense", meshgen.TET4, lambda: meshgen.random_mesh(meshgen.TET4, 900, 120, seed=10)),
]


def _np(t):
    return t.detach().cpu().numpy()


def _unpack(keys, N):
    b = mn().node_key_bits(N)
    k = _np(keys)
    k = k.view(np.uint32).astype(np.uint64) if k.dtype == np.int32 else k.view(np.uint64)
    return (k >> np.uint64(b)).astype(np.int64), (k & np.uint64((1 << b) - 1)).astype(np.int64)


def _assert_csr(got, exp, what):
    go, gi = (_np(x) for x in got)
    eo, ei = exp
    assert go.dtype == np.int64 and gi.dtype == np.int32, what
    assert np.array_equal(go, eo), f"{what}: offsets differ at {np.nonzero(go != eo)[0][:5]}"
    assert np.array_equal(gi, ei), f"{what}: indices differ at {np.nonzero(gi != ei)[0][:5]}"


# ------------------------------------------------------------------------------------------------
# row a1 / a2: pair creation
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,et,make", SMALL)
def test_row_a1_emit_node_pairs(name, et, make):
    conn, N = make()
    keys = mn().emit_node_pairs(conn.cuda(), et, N)
    a, v = _unpack(keys, N)
    ea, ev = stages.expand_node_pairs(et, conn)
    assert np.array_equal(a, ea) and np.array_equal(v, ev), name


@pytest.mark.parametrize("name,et,make", SMALL)
def test_row_a2_emit_elem_pairs(name, et, make):
    conn, N = make()
    k, v = mn().emit_elem_pairs(conn.cuda(), et, N)
    ek, ev = stages.expand_elem_pairs(et, conn)
    assert np.array_equal(_np(k), ek) and np.array_equal(_np(v), ev), name


# ------------------------------------------------------------------------------------------------
# row a3: onesweep LSD radix sort
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,et,make", SMALL)
def test_row_a3n_sort_node_pairs(name, et, make):
    conn, N = make()
    keys = mn().emit_node_pairs(conn.cuda(), et, N)
    mn().radix_sort_keys(keys, 2 * mn().node_key_bits(N))
    a, v = _unpack(keys, N)
    sa, sv = stages.sort_pairs(*stages.expand_node_pairs(et, conn))
    assert np.array_equal(a, sa) and np.array_equal(v, sv), name


@pytest.mark.parametrize("name,et,make", SMALL)
def test_row_a3e_stable_sort_elem_pairs(name, et, make):
    conn, N = make()
    k, v = mn().emit_elem_pairs(conn.cuda(), et, N)
    mn().radix_sort_pairs_u32(k, v, mn().node_key_bits(N))
    sk, sv = stages.stable_sort_by_key(*stages.expand_elem_pairs(et, conn))
    assert np.array_equal(_np(k), sk) and np.array_equal(_np(v), sv), name


@pytest.mark.parametrize("n,bits,dist", [
    (0, 20, "uniform"), (1, 20, "uniform"), (4095, 20, "uniform"), (4096, 20, "uniform"),
    (4097, 20, "uniform"), (100003, 64, "uniform"), (300001, 37, "uniform"), (200000, 33, "equal"),
    (250000, 50, "one_bucket"), (123457, 9, "skewed"), (77777, 1, "uniform"),
])
def test_row_a3_sort_adversarial_u64(n, bits, dist):
    rng = np.random.default_rng(n + bits)
    hi = (1 << bits) if bits < 64 else None
    if dist == "uniform":
        x = rng.integers(0, hi, size=n, dtype=np.uint64) if hi else rng.integers(0, 2 ** 63, size=n).astype(np.uint64) * np.uint64(2) + rng.integers(0, 2, size=n).astype(np.uint64)
    elif dist == "equal":
        x = np.full(n, (1 << (bits - 1)) + 12345, dtype=np.uint64)
    elif dist == "one_bucket":        # every key shares all digits but the lowest
        x = (np.uint64(0xABCDE) << np.uint64(20)) + rng.integers(0, 256, size=n, dtype=np.uint64)
    else:                             # 90 % of keys in one bucket
        x = np.where(rng.random(n) < 0.9, 7, rng.integers(0, 512, size=n)).astype(np.uint64)
    t = torch.from_numpy(x.view(np.int64)).cuda()
    mn().radix_sort_keys(t, bits)
    assert np.array_equal(_np(t).view(np.uint64), np.sort(x))


@pytest.mark.parametrize("n,bits", [(0, 8), (5, 3), (8191, 17), (50000, 32), (70001, 24)])
def test_row_a3_sort_u32_and_pairs(n, bits):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 1 << bits, size=n, dtype=np.uint64).astype(np.uint32)
    t = torch.from_numpy(x.view(np.int32)).cuda()
    mn().radix_sort_keys(t, bits)
    assert np.array_equal(_np(t).view(np.uint32), np.sort(x))
    # stable pairs: values record the original positions
    k = torch.from_numpy(x.view(np.int32)).cuda()
    v = torch.arange(n, dtype=torch.int32).cuda()
    mn().radix_sort_pairs_u32(k, v, bits)
    order = np.argsort(x, kind="stable")
    assert np.array_equal(_np(k).view(np.uint32), x[order]) and np.array_equal(_np(v), order)


# ------------------------------------------------------------------------------------------------
# rows a4 + a5: dedupe, run lengths, offsets
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,et,make", SMALL)
def test_row_a4_a5_unique_node(name, et, make):
    conn, N = make()
    keys = mn().emit_node_pairs(conn.cuda(), et, N)
    mn().radix_sort_keys(keys, 2 * mn().node_key_bits(N))
    got = mn().unique_node_csr(keys, N)
    k, v = stages.unique_pairs(*stages.sort_pairs(*stages.expand_node_pairs(et, conn)))
    uk, cnt = stages.reduce_by_key_ones(k)
    exp = (stages.exclusive_scan(stages.dense_counts(uk, cnt, N)), v.astype(np.int32))
    _assert_csr(got, exp, name)


@pytest.mark.parametrize("name,et,make", SMALL)
def test_row_a4_a5_elem_offsets(name, et, make):
    conn, N = make()
    k, v = mn().emit_elem_pairs(conn.cuda(), et, N)
    mn().radix_sort_pairs_u32(k, v, mn().node_key_bits(N))
    off = mn().elem_offsets(k, N)
    sk, _ = stages.stable_sort_by_key(*stages.expand_elem_pairs(et, conn))
    uk, cnt = stages.reduce_by_key_ones(sk)
    assert np.array_equal(_np(off), stages.exclusive_scan(stages.dense_counts(uk, cnt, N)))


@pytest.mark.parametrize("n", [0, 1, 31, 4096, 4097, 100000, 1000003])
def test_row_a5_exclusive_scan(n):
    rng = np.random.default_rng(n)
    c = rng.integers(0, 2000, size=n).astype(np.int32)
    got = mn().exclusive_scan(torch.from_numpy(c).cuda())
    assert np.array_equal(_np(got), stages.exclusive_scan(c))


# ------------------------------------------------------------------------------------------------
# whole path vs the std::set oracle
# ------------------------------------------------------------------------------------------------
@pytest.fixture(params=["radix", "transpose", "msd", "auto"])
def elem_path(request):
    """Forced element paths use the staged pipeline; "auto" takes the one-CTA path on small meshes."""
    mn().set_elem_path(request.param)
    yield request.param
    mn().set_elem_path("auto")


@pytest.mark.parametrize("name,et,make", SMALL)
def test_whole_path_both(name, et, make, elem_path):
    conn, N = make()
    (no, ni), (eo, ei) = mn().find_neighbors(conn.cuda(), et, N)
    _assert_csr((no, ni), oracle.node_csr(et, conn, N), name + " node " + elem_path)
    _assert_csr((eo, ei), oracle.elem_csr(et, conn, N), name + " elem " + elem_path)


@pytest.mark.parametrize("cap", [32, 96, 1 << 20])
@pytest.mark.parametrize("name,et,make", SMALL + [("kuhn_40", meshgen.TET4, lambda: meshgen.kuhn_tets(40)),
                                                  ("sphere_1000x50", meshgen.TRI3, lambda: meshgen.uv_sphere(1000, 50))])
def test_transpose_fixed_bucket_capacity(name, et, make, cap):
    """The transpose's single-read scatter into fixed-capacity chunk buckets: with a small cap some
    buckets overflow and the guarded counted path must replace the result; with a large cap (auto)
    the fixed layout is used whenever it fits.  Same CSRs either way."""
    conn, N = make()
    mn().set_elem_path("transpose")
    mn().set_chunk_cap(cap)
    try:
        (no, ni), (eo, ei) = mn().find_neighbors(conn.cuda(), et, N)
        eo2, ei2 = mn().find_elem_neighbors(conn.cuda(), et, N)
    finally:
        mn().set_chunk_cap(0)
        mn().set_elem_path("auto")
    _assert_csr((no, ni), oracle.node_csr(et, conn, N), f"{name} node cap {cap}")
    exp = oracle.elem_csr(et, conn, N)
    _assert_csr((eo, ei), exp, f"{name} elem cap {cap}")
    _assert_csr((eo2, ei2), exp, f"{name} elem-only cap {cap}")


@pytest.mark.parametrize("name,et,make", SMALL)
def test_whole_path_single_modes(name, et, make, elem_path):
    conn, N = make()
    exp = oracle.node_csr(et, conn, N)
    _assert_csr(mn().find_node_neighbors(conn.cuda(), et, N), exp, name)
    _assert_csr(mn().find_node_neighbors_sortpairs(conn.cuda(), et, N), exp, name + " sortpairs")
    _assert_csr(mn().find_elem_neighbors(conn.cuda(), et, N), oracle.elem_csr(et, conn, N), name)


@pytest.mark.parametrize("ntri", [40, 200, 20000, 30000, 60000])
def test_high_valence_fans(ntri, elem_path):
    """Node 0 and 1 of a fan see 2*ntri raw pairs: 80 (hash), 400 (block sort in shared memory),
    40000 (shared memory) and 60000 (in place in global memory) entries."""
    conn, N = meshgen.nonmanifold_fan(ntri)
    (no, ni), (eo, ei) = mn().find_neighbors(conn.cuda(), 0, N)
    _assert_csr((no, ni), oracle.node_csr(0, conn, N), f"fan{ntri}")
    _assert_csr((eo, ei), oracle.elem_csr(0, conn, N), f"fan{ntri} elem")


@pytest.mark.parametrize("name,et,make", SMALL[:6] + [SMALL[-1]])
def test_whole_path_host_buffers(name, et, make, elem_path):
    conn, N = make()
    (no, ni), (eo, ei) = mn().find_neighbors_host(conn.contiguous().pin_memory(), et, N)
    assert not no.is_cuda and no.is_pinned() and not ei.is_cuda
    _assert_csr((no, ni), oracle.node_csr(et, conn, N), name + " host node")
    _assert_csr((eo, ei), oracle.elem_csr(et, conn, N), name + " host elem")


def test_host_buffers_errors_and_empty():
    bad = torch.tensor([[0, 1, 2], [1, 2, 9]], dtype=torch.int32)
    with pytest.raises(mn().MeshError) as ei:
        mn().find_neighbors_host(bad.pin_memory(), 0, 5)
    assert (ei.value.code, ei.value.elem, ei.value.pos) == (2, 1, 2)
    (no, ni), (eo, ei_) = mn().find_neighbors_host(torch.zeros((0, 4), dtype=torch.int32), 2, 7)
    assert no.tolist() == [0] * 8 and eo.tolist() == [0] * 8 and ni.numel() == 0 and ei_.numel() == 0


def test_host_pipeline_stream_of_meshes():
    """mn_host_pipeline_*: a stream of meshes of different types and sizes with overlapping
    transfers; every ticket's CSRs equal the oracle's; tickets waited out of order; an invalid mesh
    is rejected at submit without disturbing the tickets in flight; an empty mesh."""
    pl = mn().HostPipeline()
    meshes = [(name, et, make()) for name, et, make in SMALL[:6]] + [
        ("kuhn_40", meshgen.TET4, meshgen.kuhn_tets(40))]
    tickets = []
    for name, et, (conn, N) in meshes:
        tickets.append((pl.submit(conn.contiguous().pin_memory(), et, N), name, et, conn, N))
        if len(tickets) == 3:   # an invalid mesh in the middle of the stream
            bad = torch.tensor([[0, 1, 2], [1, 2, 9]], dtype=torch.int32).pin_memory()
            with pytest.raises(mn().MeshError) as ei:
                pl.submit(bad, 0, 5)
            assert (ei.value.code, ei.value.elem, ei.value.pos) == (2, 1, 2)
    empty = pl.submit(torch.zeros((0, 4), dtype=torch.int32), 2, 7)
    for tk, name, et, conn, N in tickets[::-1]:   # reverse order
        (no, ni), (eo, ei) = pl.wait(tk)
        assert no.is_pinned() and ei.is_pinned()
        _assert_csr((no, ni), oracle.node_csr(et, conn, N), name + " pipeline node")
        _assert_csr((eo, ei), oracle.elem_csr(et, conn, N), name + " pipeline elem")
    (no, ni), (eo, ei) = pl.wait(empty)
    assert no.tolist() == [0] * 8 and eo.tolist() == [0] * 8 and ni.numel() == 0 and ei.numel() == 0
    pl.close()


def test_host_pipeline_matches_device_call_config3():
    """Config 3 (12.6 M tets) twice through the pipeline (two tickets in flight) == the
    device-buffer call, bit for bit."""
    et, conn, N = meshgen.make_config(3)
    ref = mn().find_neighbors(conn.cuda(), et, N)
    pl = mn().HostPipeline()
    h = conn.contiguous().pin_memory()
    t0, t1 = pl.submit(h, et, N), pl.submit(h, et, N)
    for tk in (t0, t1):
        got = pl.wait(tk)
        for (a, b), (c, d) in zip(got, ref):
            assert torch.equal(a, c.cpu()) and torch.equal(b, d.cpu())
    pl.close()


def test_config2_sphere_full(elem_path):
    et, conn, N = meshgen.make_config(2)
    (no, ni), (eo, ei) = mn().find_neighbors(conn.cuda(), et, N)
    _assert_csr((no, ni), oracle.node_csr(et, conn, N), "cfg2 node")
    _assert_csr((eo, ei), oracle.elem_csr(et, conn, N), "cfg2 elem")
    E = int(_np(no)[-1]) // 2
    assert N - E + conn.shape[0] == 2          # Euler on the closed sphere


# ------------------------------------------------------------------------------------------------
# edge cases and errors
# ------------------------------------------------------------------------------------------------
def test_empty_mesh_and_isolated_nodes():
    for et in (0, 1, 2, 3):
        k = meshgen.ARITY[et]
        for N in (0, 1, 17):
            c = torch.zeros((0, k), dtype=torch.int32).cuda()
            (no, ni), (eo, ei) = mn().find_neighbors(c, et, N)
            assert _np(no).tolist() == [0] * (N + 1) and ni.numel() == 0
            assert _np(eo).tolist() == [0] * (N + 1) and ei.numel() == 0
    conn = torch.tensor([[2, 5, 7]], dtype=torch.int32)
    (no, ni), _ = mn().find_neighbors(conn.cuda(), 0, 100000)
    _assert_csr((no, ni), oracle.node_csr(0, conn, 100000), "isolated")


@pytest.mark.parametrize("conn,N,et", [
    ([[0, 1, 3]], 3, 0), ([[0, 1, 1]], 3, 0), ([[0, 1, 2], [0, 1, 2], [4, 4, -1]], 5, 0),
    ([[0, 1, 2, 3]] * 5000 + [[1, 2, 3, 1]] + [[0, 9, 2, 3]], 9, 2),
    ([[0, 1, 2, 3, 4, 5, 6, 7]] * 3 + [[0, 1, 2, 3, 4, 5, 6, 6]], 8, 3),
    ([[0, 1, 2]], 0, 0),
])
def test_invalid_input_reported_like_the_oracle(conn, N, et, elem_path):
    c = torch.tensor(conn, dtype=torch.int32)
    code, elem, pos = oracle.validate(et, c, N)
    assert code != 0
    for fn in (mn().find_neighbors, mn().find_node_neighbors, mn().find_elem_neighbors):
        with pytest.raises(mn().MeshError) as ei:
            fn(c.cuda(), et, N)
        assert (ei.value.code, ei.value.elem, ei.value.pos) == (code, elem, pos)


def test_auto_elem_path_choice():
    """Config-5-like natural numbering takes the transpose, a relabelled hex the radix sort; both
    give the same CSR."""
    conn, N = meshgen.kuhn_tets(60, device="cuda")            # 1.3 M tets, coherent ids
    mn().set_elem_path("auto")
    a = mn().find_neighbors(conn, "tet4", N)
    mn().set_elem_path("radix")
    b = mn().find_neighbors(conn, "tet4", N)
    mn().set_elem_path("auto")
    for x, y in zip(a, b):
        assert torch.equal(x[0], y[0]) and torch.equal(x[1], y[1])


def test_deterministic_repeats(elem_path):
    et = meshgen.HEX8
    conn, N = _perm_hex(20, 3, 4)
    conn = conn.cuda()
    ref = mn().find_neighbors(conn, et, N)
    for _ in range(5):
        got = mn().find_neighbors(conn, et, N)
        for a, b in zip(ref, got):
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ------------------------------------------------------------------------------------------------
# full-size configs 3-5: both CSRs compared in full (memcmp) with the T-thread node-range oracle
# (SURVEY §8(c), T = host cores), plus sampled vertices vs the one-vertex form and size-free
# properties (closed-form valences, handshake, symmetry)
# ------------------------------------------------------------------------------------------------
_FULL_ORACLE = {}


def _full_oracle(cfg, et, conn_cpu, N):
    """Both oracle CSRs of a full-size config, computed once per session (T = host cores)."""
    if cfg not in _FULL_ORACLE:
        T = oracle.host_threads()
        no, ni, _ = oracle.csr_mt(oracle.NODE, et, conn_cpu, N, T)
        eo, ei, _ = oracle.csr_mt(oracle.ELEM, et, conn_cpu, N, T)
        _FULL_ORACLE[cfg] = ((no, ni), (eo, ei))
    return _FULL_ORACLE[cfg]


def _assert_full(got, exp, what):
    go, gi = (_np(x) for x in got)
    eo, ei = exp
    assert go.shape == eo.shape and np.array_equal(go, eo), f"{what}: offsets differ"
    assert gi.shape == ei.shape, f"{what}: nnz {gi.size} vs oracle {ei.size}"
    if not np.array_equal(gi, ei):
        bad = int(np.nonzero(gi != ei)[0][0])
        v = int(np.searchsorted(eo, bad, side="right") - 1)
        raise AssertionError(f"{what}: first differing index {bad} (vertex {v})")
def _sampled_check(et, conn_cpu, N, got_node, got_elem, nsample=48, seed=0):
    rng = np.random.default_rng(seed)
    sample = np.unique(np.concatenate([rng.integers(0, N, nsample), [0, N - 1, N // 2]]))
    no, ni = (_np(x) for x in got_node)
    eo, ei = (_np(x) for x in got_elem)
    exp_n = stages.node_neighbors_sample(et, conn_cpu, N, sample)
    exp_e = stages.elem_neighbors_sample(et, conn_cpu, N, sample)
    for v in sample.tolist():
        assert np.array_equal(ni[no[v]:no[v + 1]], exp_n[v]), f"node {v}"
        assert np.array_equal(ei[eo[v]:eo[v + 1]], exp_e[v]), f"elem {v}"


def _kuhn_counts(n, device):
    """Closed-form valence and element count of every node of the Kuhn n^3 mesh (torch)."""
    w = n + 1
    idx = torch.arange(w ** 3, device=device, dtype=torch.int64)
    i, j, k = idx % w, (idx // w) % w, idx // (w * w)
    val = torch.zeros_like(idx)
    for d in [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1)]:
        for s in (1, -1):
            x, y, z = i + s * d[0], j + s * d[1], k + s * d[2]
            val += ((x >= 0) & (x <= n) & (y >= 0) & (y <= n) & (z >= 0) & (z <= n)).long()
    ne = torch.zeros_like(idx)
    # tets of cell (corner offset o) containing that corner: 6 for o in {000, 111}, else 2
    for o in [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]:
        ok = (i - o[0] >= 0) & (i - o[0] < n) & (j - o[1] >= 0) & (j - o[1] < n) & (k - o[2] >= 0) & (k - o[2] < n)
        ne += ok.long() * (6 if sum(o) in (0, 3) else 2)
    return val, ne


def _symmetric(off, idx):
    rows = torch.repeat_interleave(torch.arange(off.numel() - 1, device=off.device), off[1:] - off[:-1])
    cols = idx.long()
    n = off.numel() - 1
    a = torch.sort(rows * n + cols).values
    b = torch.sort(cols * n + rows).values
    return bool(torch.equal(a, b)) and bool((rows != cols).all())


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_config(cfg, elem_path):
    et, conn, N = meshgen.make_config(cfg, device="cuda")
    (no, ni), (eo, ei) = mn().find_neighbors(conn, et, N)
    M = conn.shape[0]
    assert int(eo[-1]) == meshgen.ARITY[et] * M
    if cfg == 3:
        n = 128
        val, ne = _kuhn_counts(n, "cuda")
        assert torch.equal(no[1:] - no[:-1], val) and torch.equal(eo[1:] - eo[:-1], ne)
        assert int(no[-1]) == 2 * (3 * n * (n + 1) ** 2 + 3 * n * n * (n + 1) + n ** 3)
    else:
        n = 256
        assert int(no[-1]) == 2 * 3 * n * (n + 1) ** 2      # handshake, hex |E| = 3n(n+1)^2
        pi = torch.from_numpy(meshgen.seeded_permutation(N, 1604)).cuda()
        w = n + 1
        idx = torch.arange(N, device="cuda")
        i, j, k = idx % w, (idx // w) % w, idx // (w * w)
        inner = lambda x: (x > 0).long() + (x < n).long()
        val = inner(i) + inner(j) + inner(k)           # valence of the unpermuted node
        cnt = torch.zeros_like(no[1:])
        cnt[pi] = val
        assert torch.equal(no[1:] - no[:-1], cnt)       # permutation equivariance of valences
    assert _symmetric(no, ni)
    conn_cpu = conn.cpu()
    _sampled_check(et, conn_cpu, N, (no, ni), (eo, ei))
    ref_node, ref_elem = _full_oracle(cfg, et, conn_cpu, N)
    _assert_full((no, ni), ref_node, f"config {cfg} node CSR")
    _assert_full((eo, ei), ref_elem, f"config {cfg} elem CSR")


@pytest.mark.slow
def test_full_size_config5_single_gpu():
    et, conn, N = meshgen.make_config(5, device="cuda")
    (no, ni), (eo, ei) = mn().find_neighbors(conn, et, N)
    n = 320
    assert int(no[-1]) == 2 * (3 * n * (n + 1) ** 2 + 3 * n * n * (n + 1) + n ** 3)
    assert int(eo[-1]) == 4 * conn.shape[0]
    val, ne = _kuhn_counts(n, "cuda")
    assert torch.equal(no[1:] - no[:-1], val) and torch.equal(eo[1:] - eo[:-1], ne)
    del val, ne
    conn_cpu = conn.cpu()
    _sampled_check(et, conn_cpu, N, (no, ni), (eo, ei), nsample=24)
    del conn
    got_node = (no.cpu(), ni.cpu())
    got_elem = (eo.cpu(), ei.cpu())
    del no, ni, eo, ei
    T = oracle.host_threads()
    ro, ri, _ = oracle.csr_mt(oracle.NODE, et, conn_cpu, N, T)
    _assert_full(got_node, (ro, ri), "config 5 node CSR")
    del ro, ri, got_node
    ro, ri, _ = oracle.csr_mt(oracle.ELEM, et, conn_cpu, N, T)
    _assert_full(got_elem, (ro, ri), "config 5 elem CSR")


@pytest.mark.slow
def test_full_size_config5_lsd_paths():
    """The paper-literal node pipeline (all 2.36e9 node pairs > 2^31 as u64 keys, 7 onesweep passes
    with 54-bit look-back values and digit buckets > 2^30, then the look-back unique/compaction) and
    the LSD element path at config-5 size, bit-equal to the default path (itself memcmp-checked
    against the oracle in test_full_size_config5_single_gpu)."""
    et, conn, N = meshgen.make_config(5, device="cuda")
    ref_node, ref_elem = mn().find_neighbors(conn, et, N)
    P = 12 * conn.shape[0]
    assert P > 2 ** 31
    off, idx = mn().find_node_neighbors_sortpairs(conn, et, N)
    assert torch.equal(off, ref_node[0]) and torch.equal(idx, ref_node[1])
    del off, idx
    torch.cuda.empty_cache()
    mn().set_elem_path("radix")
    try:
        eo, ei = mn().find_elem_neighbors(conn, et, N)
    finally:
        mn().set_elem_path("auto")
    assert torch.equal(eo, ref_elem[0]) and torch.equal(ei, ref_elem[1])


# ------------------------------------------------------------------------------------------------
# memory-bounded (chunked) mode, SURVEY §8(f) row 4
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,et,make", SMALL)
@pytest.mark.parametrize("budget", [1 << 16, 1 << 20])
def test_chunked_matches_oracle(name, et, make, budget):
    conn, N = make()
    (no, ni), (eo, ei), K = mn().find_neighbors_chunked(conn.cuda(), et, N, budget)
    assert K >= 1
    _assert_csr((no, ni), oracle.node_csr(et, conn, N), f"{name} chunked node K={K}")
    _assert_csr((eo, ei), oracle.elem_csr(et, conn, N), f"{name} chunked elem K={K}")


def test_chunked_full_size_config3_bit_equal():
    et, conn, N = meshgen.make_config(3, device="cuda")
    ref = mn().find_neighbors(conn, et, N)
    budget = mn().chunk_workspace_bytes(et, conn.shape[0], N, 8)
    got = mn().find_neighbors_chunked(conn, et, N, budget)
    assert got[2] >= 8
    for a, b in zip(ref, got[:2]):
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def _traced(fn):
    m = mn()
    torch.cuda.synchronize()
    m.alloc_trace(True)
    try:
        out = fn()
        torch.cuda.synchronize()
    finally:
        trace = m.alloc_trace_take()
    return out, m.trace_peaks(trace)


@pytest.mark.parametrize("cfg", [3, 5])
def test_workspace_estimate_fidelity(cfg):
    """mn_workspace_bytes (the peak workspace the header promises) within +-10% of the peak the
    library's allocation log shows for mn_find_neighbors_both (SPEC S:L468 estimate_memory)."""
    et, conn, N = meshgen.make_config(cfg, device="cuda")
    (res, (peak, _, outb)) = _traced(lambda: mn().find_neighbors(conn, et, N))
    est = mn().workspace_bytes(et, conn.shape[0], N, 3)
    assert 0.9 * peak <= est <= 1.1 * peak, (est, peak)
    nnz = res[0][1].numel()
    assert outb >= 4 * (nnz + 4 * conn.shape[0]) + 16 * N


@pytest.mark.parametrize("cfg,budgets", [(3, [1 << 26, 1 << 28]), (5, [1 << 30, 3 << 30])])
def test_chunked_respects_budget(cfg, budgets):
    """The memory-bounded mode: the workspace the allocation log
    shows never exceeds max_workspace_bytes (outputs and the finished ranges' node-index slices
    excluded, as the header states), and the CSRs equal the unbounded call's."""
    et, conn, N = meshgen.make_config(cfg, device="cuda")
    ref = mn().find_neighbors(conn, et, N)
    (free_peak, _, _) = _traced(lambda: mn().find_neighbors(conn, et, N))[1]
    for budget in budgets:
        (got, (peak, peak_ws, _)) = _traced(lambda: mn().find_neighbors_chunked(conn, et, N, budget))
        assert peak_ws <= budget, (budget, peak_ws)
        assert peak_ws < free_peak
        assert peak - peak_ws <= 4 * ref[0][1].numel() + (1 << 20)   # only the node slices on top
        for a, b in zip(ref, got[:2]):
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        del got
    del ref


def test_chunked_splits_uneven_ranges():
    """A mesh whose incidences crowd into a few nodes (a 60,000-triangle fan plus a grid): ranges
    over budget are halved, the bound holds, the result equals the oracle."""
    fan, nf = meshgen.nonmanifold_fan(3000)
    grid, ng = meshgen.tri_grid(60, 60)
    conn = torch.cat([fan, grid + nf]).contiguous()
    N = nf + ng
    budget = 1 << 17
    ((no, ni), (eo, ei), K), (peak, peak_ws, _) = _traced(
        lambda: mn().find_neighbors_chunked(conn.cuda(), 0, N, budget))
    assert K >= 2
    assert peak_ws <= max(budget, 2 * 3000 * 4 + (1 << 16))   # single-node range: its own incidences
    _assert_csr((no, ni), oracle.node_csr(0, conn, N), "uneven chunked node")
    _assert_csr((eo, ei), oracle.elem_csr(0, conn, N), "uneven chunked elem")


@pytest.mark.parametrize("ntri", [200, 60000])
def test_chunked_fans_and_errors(ntri):
    conn, N = meshgen.nonmanifold_fan(ntri)
    (no, ni), (eo, ei), K = mn().find_neighbors_chunked(conn.cuda(), 0, N, 1 << 18)
    _assert_csr((no, ni), oracle.node_csr(0, conn, N), "fan chunked")
    _assert_csr((eo, ei), oracle.elem_csr(0, conn, N), "fan chunked elem")
    bad = torch.tensor([[0, 1, 2], [1, 2, 9]], dtype=torch.int32).cuda()
    with pytest.raises(mn().MeshError) as ei_:
        mn().find_neighbors_chunked(bad, 0, 5, 1 << 12)
    assert (ei_.value.code, ei_.value.elem, ei_.value.pos) == (2, 1, 2)


# ------------------------------------------------------------------------------------------------
# element-sharing node adjacency, SURVEY §8(f) row 3
# ------------------------------------------------------------------------------------------------
SHARED_EXTRA = [
    # hex nodes with > 30 distinct sharing neighbours: 64-slot set overflow -> block path
    ("rand_hex_dense", meshgen.HEX8, lambda: meshgen.random_mesh(meshgen.HEX8, 700, 200, seed=11)),
    ("rand_quad_dense", meshgen.QUAD4, lambda: meshgen.random_mesh(meshgen.QUAD4, 2000, 150, seed=12)),
    ("hex_grid_20", meshgen.HEX8, lambda: meshgen.hex_grid(20)),
]


@pytest.mark.parametrize("name,et,make", SMALL + SHARED_EXTRA)
def test_shared_adjacency(name, et, make, elem_path):
    conn, N = make()
    _assert_csr(mn().find_node_neighbors_shared(conn.cuda(), et, N), oracle.node_shared_csr(et, conn, N),
                name + " shared")


def test_shared_adjacency_full_size_hex():
    et, conn, N = meshgen.make_config(4, device="cuda")
    off, idx = mn().find_node_neighbors_shared(conn, et, N)
    n = 256
    w = n + 1
    i = torch.arange(N, device="cuda")
    pi = torch.from_numpy(meshgen.seeded_permutation(N, 1604)).cuda()
    ci, cj, ck = i % w, (i // w) % w, i // (w * w)
    span = lambda x: 1 + (x > 0).long() + (x < n).long()
    cnt = torch.zeros_like(off[1:])
    cnt[pi] = span(ci) * span(cj) * span(ck) - 1        # the 3x3x3 block around the node, clipped
    assert torch.equal(off[1:] - off[:-1], cnt)
    assert _symmetric(off, idx)


def test_shared_equals_edges_for_simplices_full_size():
    et, conn, N = meshgen.make_config(3, device="cuda")
    a = mn().find_node_neighbors_shared(conn, et, N)
    b = mn().find_node_neighbors(conn, et, N)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ------------------------------------------------------------------------------------------------
# one-CTA latency path for small meshes (csrc/small.cuh)
# ------------------------------------------------------------------------------------------------
SMALL_PATH = [
    ("tri_grid_32", meshgen.TRI3, lambda: meshgen.tri_grid(32, 32)),            # config 1
    ("quad_grid_20x30", meshgen.QUAD4, lambda: meshgen.quad_grid(20, 30)),
    ("kuhn_6", meshgen.TET4, lambda: meshgen.kuhn_tets(6)),
    ("hex_10_perm", meshgen.HEX8, lambda: _perm_hex(10, 3, 5)),
    ("rand_tri_dense", meshgen.TRI3, lambda: meshgen.random_mesh(meshgen.TRI3, 2500, 300, seed=21)),
    ("rand_tet_isolated", meshgen.TET4, lambda: meshgen.random_mesh(meshgen.TET4, 500, 4000, seed=22)),
    ("fan_70", meshgen.TRI3, lambda: meshgen.nonmanifold_fan(70)),
    ("fan_500_fallback", meshgen.TRI3, lambda: meshgen.nonmanifold_fan(500)),   # hub degree > 160
    ("single_tri", meshgen.TRI3, lambda: (torch.tensor([[2, 0, 1]], dtype=torch.int32), 5)),
]


@pytest.mark.parametrize("name,et,make", SMALL_PATH)
def test_small_path_matches_oracle_and_staged(name, et, make):
    conn, N = make()
    m = mn()
    m.set_elem_path("auto")
    c = conn.cuda()
    m.set_small_path(8192)
    before = m.launch_count()
    got = m.find_neighbors(c, et, N)
    launched = m.launch_count() - before
    m.set_small_path(0)
    staged = m.find_neighbors(c, et, N)
    m.set_small_path(8192)
    _assert_csr(got[0], oracle.node_csr(et, conn, N), f"{name} small node")
    _assert_csr(got[1], oracle.elem_csr(et, conn, N), f"{name} small elem")
    for a, b in zip(got, staged):
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    if "fallback" not in name:
        assert launched == 1, launched          # one kernel for both outputs
    single = m.find_node_neighbors(c, et, N), m.find_elem_neighbors(c, et, N)
    for a, b in zip(got, single):
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_small_path_validation():
    """Errors on the one-CTA path: lowest element, range before repeated node (R8)."""
    m = mn()
    conn, N = meshgen.kuhn_tets(5)
    bad = conn.clone()
    bad[300, 2] = bad[300, 0]
    bad[120, 3] = N
    bad[120, 1] = bad[120, 0]
    with pytest.raises(m.MeshError) as ei:
        m.find_neighbors(bad.cuda(), "tet4", N)
    assert (ei.value.code, ei.value.elem, ei.value.pos) == (m.MN_ERR_INDEX_OUT_OF_RANGE, 120, 3)
    assert oracle.validate(meshgen.TET4, bad, N) == (oracle.ERR_RANGE, 120, 3)
