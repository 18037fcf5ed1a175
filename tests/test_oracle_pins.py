"""Pins for the oracle (oracle/), CPU only.

Every check here compares the oracle with something that is NOT the oracle: values from the
SPEC/paper worked examples (tests/golden/), brute force from the definitions on tiny meshes,
closed forms of the structured generators, Euler / handshake / symmetry invariants, and the
library special case "element CSR = transpose of the incidence matrix B, simplicial node CSR =
pattern(B^T B) - I" (scipy.sparse).  Each pin names the mistake it catches.
"""
import itertools

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import meshgen
import oracle
from oracle import stages

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")

BOTH_NODE = [("set", oracle.node_csr), ("stages", stages.node_csr)]
BOTH_ELEM = [("set", oracle.elem_csr), ("stages", stages.elem_csr)]


def _np(conn):
    return conn.numpy() if isinstance(conn, torch.Tensor) else np.asarray(conn, dtype=np.int32)


def _slices(offsets, indices):
    return [indices[offsets[v]:offsets[v + 1]].tolist() for v in range(len(offsets) - 1)]


# ------------------------------------------------------------------------------------------
# brute force from the definitions (tiny meshes). The edge relation is derived WITHOUT the
# oracle's tables: simplices -> any two nodes of the element; quad -> ring neighbours;
# hex -> local VTK corner coordinates at Hamming distance 1.
# ------------------------------------------------------------------------------------------
_VTK_HEX_XYZ = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]


def _is_edge(etype, i, j):
    if etype in (meshgen.TRI3, meshgen.TET4):
        return i != j
    if etype == meshgen.QUAD4:
        return (i - j) % 4 in (1, 3)
    a, b = _VTK_HEX_XYZ[i], _VTK_HEX_XYZ[j]
    return sum(x != y for x, y in zip(a, b)) == 1


def brute_node(etype, conn, N):
    conn = _np(conn).reshape(-1, meshgen.ARITY[etype])
    adj = [[] for _ in range(N)]
    for u in range(N):
        for v in range(N):
            if u == v:
                continue
            hit = False
            for row in conn:
                for i, j in itertools.permutations(range(len(row)), 2):
                    if row[i] == u and row[j] == v and _is_edge(etype, i, j):
                        hit = True
                        break
                if hit:
                    break
            if hit:
                adj[u].append(v)
    return adj


def brute_elem(etype, conn, N):
    conn = _np(conn).reshape(-1, meshgen.ARITY[etype])
    return [[e for e in range(len(conn)) if v in conn[e].tolist()] for v in range(N)]


# ------------------------------------------------------------------------------------------
# golden worked examples
# ------------------------------------------------------------------------------------------
def test_golden_pairs(golden):
    for case in golden["node_pairs"]:
        k, v = stages.expand_node_pairs(case["etype"], np.array(case["conn"]))
        if "keys" in case:
            assert k.tolist() == case["keys"], case["cite"]
            assert v.tolist() == case["values"], case["cite"]
        if "count" in case:
            assert len(k) == case["count"], case["cite"]
            for a, b, mult in case["pair_multiplicity"]:
                assert int(np.sum((k == a) & (v == b))) == mult, case["cite"]
    for case in golden["elem_pairs"]:
        k, v = stages.expand_elem_pairs(case["etype"], np.array(case["conn"]))
        assert k.tolist() == case["keys"] and v.tolist() == case["values"], case["cite"]


def test_golden_primitives(golden):
    for c in golden["sort_pairs"]:
        k, v = stages.sort_pairs(np.array(c["keys"]), np.array(c["values"]))
        assert k.tolist() == c["sorted_keys"] and v.tolist() == c["sorted_values"], c["cite"]
    for c in golden["exclusive_scan"]:
        assert stages.exclusive_scan(c["counts"]).tolist() == c["offsets"], c["cite"]
    for c in golden["reduce_by_key_ones"]:
        u, n = stages.reduce_by_key_ones(np.array(c["keys"]))
        assert u.tolist() == c["unique"] and n.tolist() == c["counts"], c["cite"]
    for c in golden["first_positions_by_key"]:
        u, f = stages.first_positions_by_key(np.array(c["keys"]))
        assert u.tolist() == c["unique"] and f.tolist() == c["first"], c["cite"]


def _check_csr_case(case, fn):
    conn = np.array(case["conn"], dtype=np.int32).reshape(-1, meshgen.ARITY[case["etype"]])
    off, idx = fn(case["etype"], conn, case["num_nodes"])
    if "offsets" in case:
        assert off.tolist() == case["offsets"], case["cite"]
        assert idx.tolist() == case["indices"], case["cite"]
    for v, s in case.get("slices", {}).items():
        v = int(v)
        assert idx[off[v]:off[v + 1]].tolist() == s, case["cite"]


@pytest.mark.parametrize("name,fn", BOTH_NODE)
def test_golden_node_csr(golden, name, fn):
    for case in golden["node_csr"]:
        _check_csr_case(case, fn)


@pytest.mark.parametrize("name,fn", BOTH_ELEM)
def test_golden_elem_csr(golden, name, fn):
    for case in golden["elem_csr"]:
        _check_csr_case(case, fn)


def test_golden_validation(golden):
    for case in golden["validation"]:
        conn = np.array(case["conn"], dtype=np.int32)
        code, elem, pos = oracle.validate(case["etype"], conn, case["num_nodes"])
        assert code == case["code"], case["cite"]
        if code:
            assert (elem, pos) == (case["elem"], case["pos"]), case["cite"]
            with pytest.raises(oracle.OracleMeshError) as ei:
                oracle.node_csr(case["etype"], conn, case["num_nodes"])
            assert (ei.value.code, ei.value.elem, ei.value.pos) == (code, elem, pos)


# ------------------------------------------------------------------------------------------
# brute force on tiny meshes of every element type
# ------------------------------------------------------------------------------------------
TINY = [
    ("tri_grid_2x3", lambda: meshgen.tri_grid(2, 3)),
    ("quad_grid_2x2", lambda: meshgen.quad_grid(2, 2)),
    ("kuhn_1", lambda: meshgen.kuhn_tets(1)),
    ("hex_2", lambda: meshgen.hex_grid(2)),
    ("sphere_5x3", lambda: meshgen.uv_sphere(5, 3)),
    ("fan3", lambda: meshgen.nonmanifold_fan(3)),
    ("rand_tri", lambda: meshgen.random_mesh(meshgen.TRI3, 9, 11, seed=1)),
    ("rand_quad", lambda: meshgen.random_mesh(meshgen.QUAD4, 6, 10, seed=2)),
    ("rand_tet", lambda: meshgen.random_mesh(meshgen.TET4, 7, 9, seed=3)),
    ("rand_hex", lambda: meshgen.random_mesh(meshgen.HEX8, 3, 14, seed=4)),
]
TINY_TYPES = {"tri_grid_2x3": 0, "quad_grid_2x2": 1, "kuhn_1": 2, "hex_2": 3, "sphere_5x3": 0,
              "fan3": 0, "rand_tri": 0, "rand_quad": 1, "rand_tet": 2, "rand_hex": 3}


@pytest.mark.parametrize("name,make", TINY)
def test_brute_force(name, make):
    conn, N = make()
    et = TINY_TYPES[name]
    bn, be = brute_node(et, conn, N), brute_elem(et, conn, N)
    for _, fn in BOTH_NODE:
        assert _slices(*fn(et, conn, N)) == bn, name
    for _, fn in BOTH_ELEM:
        assert _slices(*fn(et, conn, N)) == be, name


# ------------------------------------------------------------------------------------------
# closed forms of the structured generators
# ------------------------------------------------------------------------------------------
def _grid_closed_form_tri(r, c):
    w = c + 1
    nid = lambda i, j: i + w * j
    adj, inc = [], []
    for j in range(r + 1):
        for i in range(c + 1):
            a = []
            for di, dj in [(1, 0), (0, 1), (1, 1), (-1, 0), (0, -1), (-1, -1)]:
                if 0 <= i + di <= c and 0 <= j + dj <= r:
                    a.append(nid(i + di, j + dj))
            adj.append(sorted(a))
            e = []
            # (cell offset, which triangle of the cell) that contain corner (i, j)
            for (ci, cj, t) in [(i, j, 0), (i, j, 1), (i - 1, j, 0), (i - 1, j - 1, 0),
                                (i - 1, j - 1, 1), (i, j - 1, 1)]:
                if 0 <= ci < c and 0 <= cj < r:
                    e.append(2 * (ci + c * cj) + t)
            inc.append(sorted(e))
    return adj, inc


def _kuhn_closed_form(n):
    w = n + 1
    nid = lambda i, j, k: i + w * (j + w * k)
    dirs = [d for d in itertools.product((0, 1), repeat=3) if any(d)]
    adj, inc = [], []
    for k in range(w):
        for j in range(w):
            for i in range(w):
                a = set()
                for d in dirs:
                    for s in (1, -1):
                        x, y, z = i + s * d[0], j + s * d[1], k + s * d[2]
                        if 0 <= x <= n and 0 <= y <= n and 0 <= z <= n:
                            a.add(nid(x, y, z))
                adj.append(sorted(a))
                e = []
                for o in itertools.product((0, 1), repeat=3):
                    ci, cj, ck = i - o[0], j - o[1], k - o[2]
                    if not (0 <= ci < n and 0 <= cj < n and 0 <= ck < n):
                        continue
                    cell = ci + n * (cj + n * ck)
                    axes = {ax for ax in range(3) if o[ax]}
                    for p, perm in enumerate(meshgen.KUHN_PERMS):
                        # tet p's corners: 0, e_p0, e_p0 + e_p1, (1,1,1)
                        corners = [set(), {perm[0]}, {perm[0], perm[1]}, {0, 1, 2}]
                        if axes in corners:
                            e.append(6 * cell + p)
                inc.append(sorted(e))
    return adj, inc


def _hex_closed_form(n):
    w = n + 1
    nid = lambda i, j, k: i + w * (j + w * k)
    adj, inc = [], []
    for k in range(w):
        for j in range(w):
            for i in range(w):
                a = []
                for d in [(1, 0, 0), (0, 1, 0), (0, 0, 1), (-1, 0, 0), (0, -1, 0), (0, 0, -1)]:
                    x, y, z = i + d[0], j + d[1], k + d[2]
                    if 0 <= x <= n and 0 <= y <= n and 0 <= z <= n:
                        a.append(nid(x, y, z))
                adj.append(sorted(a))
                e = []
                for o in itertools.product((0, 1), repeat=3):
                    ci, cj, ck = i - o[0], j - o[1], k - o[2]
                    if 0 <= ci < n and 0 <= cj < n and 0 <= ck < n:
                        e.append(ci + n * (cj + n * ck))
                inc.append(sorted(e))
    return adj, inc


@pytest.mark.parametrize("name,fn", BOTH_NODE)
def test_closed_form_tri_grid(name, fn):
    r, c = 7, 9
    conn, N = meshgen.tri_grid(r, c)
    adj, inc = _grid_closed_form_tri(r, c)
    assert _slices(*fn(meshgen.TRI3, conn, N)) == adj
    efn = oracle.elem_csr if name == "set" else stages.elem_csr
    assert _slices(*efn(meshgen.TRI3, conn, N)) == inc


@pytest.mark.parametrize("name,fn", BOTH_NODE)
def test_closed_form_kuhn(name, fn):
    n = 5
    conn, N = meshgen.kuhn_tets(n)
    adj, inc = _kuhn_closed_form(n)
    assert _slices(*fn(meshgen.TET4, conn, N)) == adj
    efn = oracle.elem_csr if name == "set" else stages.elem_csr
    assert _slices(*efn(meshgen.TET4, conn, N)) == inc


@pytest.mark.parametrize("name,fn", BOTH_NODE)
def test_closed_form_hex(name, fn):
    n = 4
    conn, N = meshgen.hex_grid(n)
    adj, inc = _hex_closed_form(n)
    assert _slices(*fn(meshgen.HEX8, conn, N)) == adj
    efn = oracle.elem_csr if name == "set" else stages.elem_csr
    assert _slices(*efn(meshgen.HEX8, conn, N)) == inc


def test_closed_form_quad_grid():
    r, c = 4, 6
    conn, N = meshgen.quad_grid(r, c)
    w = c + 1
    off, idx = oracle.node_csr(meshgen.QUAD4, conn, N)
    eoff, eidx = oracle.elem_csr(meshgen.QUAD4, conn, N)
    for j in range(r + 1):
        for i in range(c + 1):
            v = i + w * j
            exp = sorted(x + w * y for x, y in [(i + 1, j), (i - 1, j), (i, j + 1), (i, j - 1)]
                         if 0 <= x <= c and 0 <= y <= r)
            assert idx[off[v]:off[v + 1]].tolist() == exp
            expe = sorted(x + c * y for x, y in [(i, j), (i - 1, j), (i, j - 1), (i - 1, j - 1)]
                          if 0 <= x < c and 0 <= y < r)
            assert eidx[eoff[v]:eoff[v + 1]].tolist() == expe


def test_interior_valences():
    """north_star: interior valence 6 (Freudenthal tri) / 14 (Kuhn); element counts 6 / 24 / 8."""
    for (conn, N), et, lo, hi, nv, ne in [
        (meshgen.tri_grid(6, 6), meshgen.TRI3, 1, 5, 6, 6),
    ]:
        off, _ = oracle.node_csr(et, conn, N)
        eoff, _ = oracle.elem_csr(et, conn, N)
        for j in range(lo, hi + 1):
            for i in range(lo, hi + 1):
                v = i + 7 * j
                assert off[v + 1] - off[v] == nv and eoff[v + 1] - eoff[v] == ne
    for make, et, nv, ne in [(meshgen.kuhn_tets, meshgen.TET4, 14, 24),
                             (meshgen.hex_grid, meshgen.HEX8, 6, 8)]:
        n = 4
        conn, N = make(n)
        off, _ = oracle.node_csr(et, conn, N)
        eoff, _ = oracle.elem_csr(et, conn, N)
        w = n + 1
        for k in range(1, n):
            for j in range(1, n):
                for i in range(1, n):
                    v = i + w * (j + w * k)
                    assert off[v + 1] - off[v] == nv and eoff[v + 1] - eoff[v] == ne


# ------------------------------------------------------------------------------------------
# invariants: handshake with closed-form |E|, Euler on spheres, symmetry
# ------------------------------------------------------------------------------------------
def test_handshake_closed_form_edges():
    r, c = 10, 10
    conn, N = meshgen.tri_grid(r, c)
    off, _ = oracle.node_csr(meshgen.TRI3, conn, N)
    # |E| = r(c+1) + c(r+1) + rc (S:L74's "340" is an arithmetic slip, it is 320)
    assert off[-1] == 2 * (r * (c + 1) + c * (r + 1) + r * c) == 2 * 320
    n = 4
    conn, N = meshgen.kuhn_tets(n)
    off, _ = oracle.node_csr(meshgen.TET4, conn, N)
    assert off[-1] == 2 * (3 * n * (n + 1) ** 2 + 3 * n * n * (n + 1) + n ** 3)
    conn, N = meshgen.hex_grid(n)
    off, _ = oracle.node_csr(meshgen.HEX8, conn, N)
    assert off[-1] == 2 * (3 * n * (n + 1) ** 2)
    eoff, _ = oracle.elem_csr(meshgen.HEX8, conn, N)
    assert eoff[-1] == 8 * conn.shape[0]


@pytest.mark.parametrize("nlon,nrings", [(3, 1), (8, 5), (40, 21)])
def test_sphere_euler(nlon, nrings):
    conn, N = meshgen.uv_sphere(nlon, nrings)
    F = conn.shape[0]
    off, idx = oracle.node_csr(meshgen.TRI3, conn, N)
    E = off[-1] // 2
    assert N - E + F == 2                      # Euler, genus 0
    assert 2 * E == 3 * F                      # closed 2-manifold: every edge in two triangles
    k, v = stages.expand_node_pairs(meshgen.TRI3, conn)
    pairs = k.astype(np.int64) * N + v
    _, mult = np.unique(pairs, return_counts=True)
    assert np.all(mult == 2)                   # every directed pair created exactly twice
    assert off[1] - off[0] == nlon and off[-1] - off[-2] == nlon   # poles


@pytest.mark.parametrize("make,et", [(lambda: meshgen.kuhn_tets(3), 2), (lambda: meshgen.hex_grid(3), 3),
                                     (lambda: meshgen.random_mesh(0, 200, 60, seed=7), 0)])
def test_symmetry_ascending_no_self(make, et):
    conn, N = make()
    off, idx = oracle.node_csr(et, conn, N)
    s = _slices(off, idx)
    for v, lst in enumerate(s):
        assert v not in lst
        assert all(a < b for a, b in zip(lst, lst[1:]))
        for u in lst:
            assert v in s[u]


# ------------------------------------------------------------------------------------------
# library special case: incidence matrix B (M x N)
# ------------------------------------------------------------------------------------------
def _incidence(conn, N):
    conn = _np(conn)
    M, k = conn.shape
    rows = np.repeat(np.arange(M), k)
    return sp.csr_matrix((np.ones(M * k, dtype=np.int64), (rows, conn.reshape(-1))), shape=(M, N))


@pytest.mark.parametrize("make,et", [(lambda: meshgen.kuhn_tets(3), 2), (lambda: meshgen.tri_grid(5, 4), 0),
                                     (lambda: meshgen.random_mesh(2, 150, 40, seed=11), 2),
                                     (lambda: meshgen.random_mesh(0, 150, 40, seed=12), 0)])
def test_incidence_matrix(make, et):
    conn, N = make()
    B = _incidence(conn, N)
    Bt = sp.csr_matrix(B.T)
    Bt.sort_indices()
    eoff, eidx = oracle.elem_csr(et, conn, N)
    assert eoff.tolist() == Bt.indptr.tolist() and eidx.tolist() == Bt.indices.tolist()
    A = (B.T @ B).tolil()
    A.setdiag(0)
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    A.sort_indices()
    off, idx = oracle.node_csr(et, conn, N)
    assert off.tolist() == A.indptr.tolist() and idx.tolist() == A.indices.tolist()


def test_incidence_hex_is_not_pattern():
    """For hexes the node relation is edges only: pattern(B^T B) - I must be strictly larger."""
    conn, N = meshgen.hex_grid(2)
    off, _ = oracle.node_csr(meshgen.HEX8, conn, N)
    B = _incidence(conn, N)
    A = (B.T @ B).tolil()
    A.setdiag(0)
    assert sp.csr_matrix(A).nnz > off[-1]


# ------------------------------------------------------------------------------------------
# permutation equivariance (config-4 style relabelled hex)
# ------------------------------------------------------------------------------------------
def test_permutation_equivariance():
    n = 4
    conn, N = meshgen.hex_grid(n)
    pconn = meshgen.relabel(conn, N, 1604, 4689)
    pi = meshgen.seeded_permutation(N, 1604)
    sigma = meshgen.seeded_permutation(conn.shape[0], 4689)
    sinv = np.argsort(sigma)
    a0 = _slices(*oracle.node_csr(3, conn, N))
    a1 = _slices(*oracle.node_csr(3, pconn, N))
    e0 = _slices(*oracle.elem_csr(3, conn, N))
    e1 = _slices(*oracle.elem_csr(3, pconn, N))
    for v in range(N):
        assert a1[pi[v]] == sorted(int(pi[u]) for u in a0[v])
        assert e1[pi[v]] == sorted(int(sinv[e]) for e in e0[v])


# ------------------------------------------------------------------------------------------
# edge cases
# ------------------------------------------------------------------------------------------
def test_empty_and_isolated():
    empty = np.zeros((0, 3), dtype=np.int32)
    for fn in (oracle.node_csr, oracle.elem_csr, stages.node_csr, stages.elem_csr):
        off, idx = fn(0, empty, 0)
        assert off.tolist() == [0] and idx.size == 0
        off, idx = fn(0, empty, 5)
        assert off.tolist() == [0] * 6 and idx.size == 0
    conn = np.array([[2, 5, 7]], dtype=np.int32)
    off, idx = oracle.node_csr(0, conn, 10)
    assert off.tolist() == [0, 0, 0, 2, 2, 2, 4, 4, 6, 6, 6]
    assert idx.tolist() == [5, 7, 2, 7, 2, 5]


def test_seeded_permutation_is_permutation():
    p = meshgen.seeded_permutation(1000, 1604)
    assert sorted(p.tolist()) == list(range(1000))
    assert not np.array_equal(p, np.arange(1000))
    assert np.array_equal(p, meshgen.seeded_permutation(1000, 1604))


def test_generator_sizes():
    """Config shapes from BASELINE.json / SURVEY §8.0 (closed forms of the recipes)."""
    conn, N = meshgen.tri_grid(32, 32)
    assert conn.shape == (2048, 3) and N == 1089
    conn, N = meshgen.uv_sphere(1000, 501)
    assert conn.shape == (1002000, 3) and N == 501002
    conn, N = meshgen.kuhn_tets(8)
    assert conn.shape == (6 * 512, 4) and N == 729
    assert meshgen.kuhn_tets(8, cell_begin=100, cell_end=200)[0].equal(conn[600:1200])


# ------------------------------------------------------------------------------------------------
# element-sharing node adjacency: pattern(B^T B) - I for every element type,
# brute force from its definition, and equal to the edge adjacency for simplices
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("make,et", [(lambda: meshgen.hex_grid(3), 3), (lambda: meshgen.quad_grid(4, 5), 1),
                                     (lambda: meshgen.random_mesh(3, 60, 80, seed=13), 3),
                                     (lambda: meshgen.random_mesh(1, 90, 60, seed=14), 1)])
def test_shared_adjacency_is_incidence_pattern(make, et):
    conn, N = make()
    B = _incidence(conn, N)
    A = (B.T @ B).tolil()
    A.setdiag(0)
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    A.sort_indices()
    off, idx = oracle.node_shared_csr(et, conn, N)
    assert off.tolist() == A.indptr.tolist() and idx.tolist() == A.indices.tolist()


def test_shared_adjacency_brute_force_and_simplices():
    conn, N = meshgen.random_mesh(meshgen.HEX8, 4, 14, seed=15)
    c = _np(conn)
    brute = [sorted({int(x) for row in c if v in row.tolist() for x in row.tolist() if x != v}) for v in range(N)]
    assert _slices(*oracle.node_shared_csr(3, conn, N)) == brute
    for make, et in [(lambda: meshgen.kuhn_tets(3), 2), (lambda: meshgen.tri_grid(4, 3), 0)]:
        conn, N = make()
        a, b = oracle.node_shared_csr(et, conn, N), oracle.node_csr(et, conn, N)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # interior hex node: 26 sharing neighbours (the 3x3x3 block); interior quad node: 8
    n = 4
    conn, N = meshgen.hex_grid(n)
    off, _ = oracle.node_shared_csr(3, conn, N)
    v = 2 + 5 * (2 + 5 * 2)
    assert off[v + 1] - off[v] == 26
    conn, N = meshgen.quad_grid(4, 4)
    off, _ = oracle.node_shared_csr(1, conn, N)
    assert off[12 + 1] - off[12] == 8
