"""GPU parity of the polygon / mixed-arity path (mn_find_poly_neighbors)
against the oracle (oracle.poly_*), bit-exact: ring-edge node CSR, element CSR, element-sharing
node CSR."""
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
        pytest.skip("needs a GPU")
    from paper_1604_04689_b200 import build
    build.build()


def mn():
    import paper_1604_04689_b200 as m
    return m


def _eq(got, exp, what):
    go, gi = got[0].cpu().numpy(), got[1].cpu().numpy()
    eo, ei = exp
    assert np.array_equal(go, eo), f"{what}: offsets differ"
    assert np.array_equal(gi, ei), f"{what}: indices differ"


def _fan(k, n):
    """n polygons of arity k sharing node 0 (node 0 has 2n ring neighbours: giant path)."""
    rings = [[0] + [1 + (k - 1) * t + q for q in range(k - 1)] for t in range(n)]
    off = np.cumsum([0] + [len(r) for r in rings])
    return torch.from_numpy(off.astype(np.int64)), torch.from_numpy(np.concatenate(rings).astype(np.int32)), \
        1 + (k - 1) * n


CASES = [
    ("mixed_1x1", lambda: meshgen.poly_mixed_grid(1, 1, 0)),
    ("mixed_37x53", lambda: meshgen.poly_mixed_grid(37, 53, 1604)),
    ("mixed_150x90_perm", lambda: (lambda o, i, n: (*meshgen.poly_relabel(o, i, n, 5, 6), n))(
        *meshgen.poly_mixed_grid(150, 90, 7))),
    ("honeycomb_40x33", lambda: meshgen.honeycomb(40, 33)),
    ("rand_3_7", lambda: meshgen.random_poly(3000, 2000, 3, 7, 1)),
    ("rand_3_12_dense", lambda: meshgen.random_poly(2000, 150, 3, 12, 2)),      # giants in both modes
    ("rand_big_rings", lambda: meshgen.random_poly(300, 5000, 20, 60, 3)),      # shared raw > 24 per incidence
    ("fan_5x40", lambda: _fan(5, 40)),
    ("fan_3x3000", lambda: _fan(3, 3000)),
    ("tri_as_poly", lambda: (*meshgen.poly_from_conn(meshgen.tri_grid(31, 44)[0]), 32 * 45)),
    ("quad_as_poly", lambda: (*meshgen.poly_from_conn(meshgen.quad_grid(20, 17)[0]), 21 * 18)),
]


@pytest.mark.parametrize("name,make", CASES)
def test_poly_parity(name, make):
    off, idx, N = make()
    node, elem, shared = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, node=True, elem=True, shared=True)
    _eq(node, oracle.poly_node_csr(off, idx, N), name + " node")
    _eq(elem, oracle.poly_elem_csr(off, idx, N), name + " elem")
    _eq(shared, oracle.poly_shared_csr(off, idx, N), name + " shared")


@pytest.mark.parametrize("cap", [0, 32, 96])
@pytest.mark.parametrize("name,make", CASES)
def test_poly_chunk_path(name, make, cap):
    """Node + element outputs (no element-sharing CSR) take the chunk-bucketed transpose: fixed
    capacity buckets (cap 0 = auto), with small caps forcing the guarded counted fallback."""
    off, idx, N = make()
    mn().set_chunk_cap(cap)
    try:
        node, elem, _ = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, node=True, elem=True)
        elem_only = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, node=False, elem=True)[1]
        node_only = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, node=True, elem=False)[0]
    finally:
        mn().set_chunk_cap(0)
    en, ee = oracle.poly_node_csr(off, idx, N), oracle.poly_elem_csr(off, idx, N)
    _eq(node, en, f"{name} node cap {cap}")
    _eq(node_only, en, f"{name} node-only cap {cap}")
    _eq(elem, ee, f"{name} elem cap {cap}")
    _eq(elem_only, ee, f"{name} elem-only cap {cap}")


@pytest.mark.parametrize("sel", [(True, False, False), (False, True, False), (False, False, True),
                                 (True, False, True)])
def test_output_selection(sel):
    off, idx, N = meshgen.poly_mixed_grid(33, 29, 9)
    outs = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, *sel)
    exp = (oracle.poly_node_csr, oracle.poly_elem_csr, oracle.poly_shared_csr)
    for want, got, fn in zip(sel, outs, exp):
        if want:
            _eq(got, fn(off, idx, N), fn.__name__)
        else:
            assert got is None


def test_fixed_types_agree():
    """A TRI3 / QUAD4 mesh through the polygon path equals the fixed-type path."""
    for make, et in ((lambda: meshgen.tri_grid(60, 41), meshgen.TRI3), (lambda: meshgen.quad_grid(50, 37), meshgen.QUAD4)):
        conn, N = make()
        off, idx = meshgen.poly_from_conn(conn)
        node, elem, shared = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, True, True, True)
        (no, ni), (eo, ei) = mn().find_neighbors(conn.cuda(), et, N)
        so, si = mn().find_node_neighbors_shared(conn.cuda(), et, N)
        for a, b in ((node, (no, ni)), (elem, (eo, ei)), (shared, (so, si))):
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_empty_and_isolated():
    off = torch.zeros(1, dtype=torch.int64, device="cuda")
    idx = torch.zeros(0, dtype=torch.int32, device="cuda")
    node, elem, shared = mn().find_poly_neighbors(off, idx, 5, True, True, True)
    for o, i in (node, elem, shared):
        assert o.tolist() == [0] * 6 and i.numel() == 0
    node, elem, shared = mn().find_poly_neighbors(off, idx, 0, True, True, True)
    assert node[0].tolist() == [0]


def _P(rings):
    off = torch.tensor(np.cumsum([0] + [len(r) for r in rings]), dtype=torch.int64)
    idx = torch.tensor([x for r in rings for x in r], dtype=torch.int32)
    return off, idx


@pytest.mark.parametrize("rings,N", [
    ([[0, 1, 2], [5, 9], [0, 9, 9]], 10),          # arity error first (R18)
    ([[0, 1, 2, 3], [0, 9, 9], [7, 8]], 4),          # range error in element 1, arity error later
    ([[0, 1, 2, 3, 2, 9]], 10),                      # repeated node at position 4
    ([[0, 1, 2], [3, 4, 5, 3]], 6),
    ([[0, 1, 2]], 3),
])
def test_validation_matches_oracle(rings, N):
    off, idx = _P(rings)
    code, e, p = oracle.poly_validate(off, idx, N)
    m = mn()
    if code == oracle.OK:
        m.find_poly_neighbors(off.cuda(), idx.cuda(), N)
        return
    want = {oracle.ERR_RANGE: m.MN_ERR_INDEX_OUT_OF_RANGE, oracle.ERR_DEGENERATE: m.MN_ERR_DEGENERATE,
            oracle.ERR_ARITY: m.MN_ERR_ARITY}[code]
    for sel in ((True, True, True), (True, True, False), (False, True, False)):   # counted / chunk paths
        with pytest.raises(m.MeshError) as ei:
            m.find_poly_neighbors(off.cuda(), idx.cuda(), N, *sel)
        assert (ei.value.code, ei.value.elem, ei.value.pos) == (want, e, p), sel


def test_bad_offsets():
    m = mn()
    off = torch.tensor([0, 3, 5], dtype=torch.int64, device="cuda")     # off[M] != len(idx)
    idx = torch.arange(6, dtype=torch.int32, device="cuda")
    with pytest.raises(m.MeshError) as ei:
        m.find_poly_neighbors(off, idx, 6)
    assert ei.value.code == m.MN_ERR_INVALID_ARG
    off = torch.tensor([1, 4, 7], dtype=torch.int64, device="cuda")     # off[0] != 0
    idx = torch.arange(7, dtype=torch.int32, device="cuda")
    with pytest.raises(m.MeshError) as ei:
        m.find_poly_neighbors(off, idx, 7)
    assert ei.value.code == m.MN_ERR_INVALID_ARG


def test_deterministic():
    off, idx, N = meshgen.random_poly(5000, 900, 3, 9, 4)
    a = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, True, True, True)
    b = mn().find_poly_neighbors(off.cuda(), idx.cuda(), N, True, True, True)
    for x, y in zip(a, b):
        assert torch.equal(x[0], y[0]) and torch.equal(x[1], y[1])


def test_full_size_poly_config():
    """Config 6 (mixed grid 8192^2, the polygon bench workload): sampled nodes against the oracle's
    single-vertex form, the closed-form edge count, symmetry."""
    off, idx, N = meshgen.make_poly_config(6, device="cuda")
    node, elem, shared = mn().find_poly_neighbors(off, idx, N, True, True, True)
    r = c = 8192
    split = off.numel() - 1 - r * c
    assert int(node[0][-1]) == 2 * (r * (c + 1) + c * (r + 1) + split)
    assert int(elem[0][-1]) == idx.numel()
    rng = np.random.default_rng(6)
    sample = np.unique(np.concatenate([rng.integers(0, N, 40), [0, N - 1, c, N - 1 - c]]))
    exp = stages.poly_neighbors_sample(off, idx, N, sample)
    for (o, i), j in ((node, 0), (elem, 1), (shared, 2)):
        oc = o.cpu().numpy()
        for v in sample.tolist():
            got = i[oc[v]:oc[v + 1]].cpu().numpy()
            assert np.array_equal(got, exp[v][j]), (j, v)


def test_ingest_then_find():
    """OFF/OBJ text -> native parser -> polygon path, against the oracle on the generator's arrays."""
    off, idx, N = meshgen.poly_mixed_grid(40, 31, 12)
    o, i = off.numpy(), idx.numpy()
    text = "OFF\n%d %d 0\n" % (N, len(o) - 1) + "0 0 0\n" * N + \
        "".join("%d %s\n" % (o[e + 1] - o[e], " ".join(map(str, i[o[e]:o[e + 1]]))) for e in range(len(o) - 1))
    po, pi, pn, k = mn().load_off(text.encode())
    node, elem, shared = mn().find_poly_neighbors(po.cuda(), pi.cuda(), pn, True, True, True)
    _eq(node, oracle.poly_node_csr(off, idx, N), "node")
    _eq(elem, oracle.poly_elem_csr(off, idx, N), "elem")
    _eq(shared, oracle.poly_shared_csr(off, idx, N), "shared")
