"""Pins of the polygon / mixed-arity oracle (oracle.poly_*).

Each pin checks the oracle against something other than itself:
* reduction: a polygon mesh whose rings all have 3 (4) nodes is a TRI3 (QUAD4) mesh, whose oracle is
  pinned separately (tests/test_oracle_pins.py: closed forms, SPEC examples, brute force);
* brute force: pure-Python ring-edge sets on tiny random polygon soups;
* closed forms: the mixed grid's edge count r(c+1) + c(r+1) + #split cells, the honeycomb's
  Euler characteristic V - E + F = 1 (a disk) and interior valence 3;
* linear algebra: element-sharing adjacency = pattern(B^T B) - I, B the element x node incidence;
* validation: SPEC validate_mesh examples and reading R18 (arity, then range, then
  repeated node; lowest element first).
"""
import numpy as np
import pytest

import meshgen
import oracle


def _lists(off, idx):
    return [idx[off[v]:off[v + 1]].tolist() for v in range(len(off) - 1)]


def _brute(off, idx, N, mode):
    off, idx = np.asarray(off), np.asarray(idx)
    out = [set() for _ in range(N)]
    inc = [[] for _ in range(N)]
    for e in range(len(off) - 1):
        ring = idx[off[e]:off[e + 1]].tolist()
        k = len(ring)
        for p, a in enumerate(ring):
            inc[a].append(e)
            if mode == "node":
                out[a].add(ring[(p + 1) % k])
                out[a].add(ring[(p - 1) % k])
            else:
                out[a].update(x for x in ring if x != a)
    if mode == "elem":
        return inc
    return [sorted(s) for s in out]


@pytest.mark.parametrize("make,et", [(lambda: meshgen.tri_grid(7, 5), meshgen.TRI3),
                                     (lambda: meshgen.quad_grid(6, 9), meshgen.QUAD4),
                                     (lambda: meshgen.uv_sphere(12, 7), meshgen.TRI3),
                                     (lambda: meshgen.random_mesh(meshgen.QUAD4, 300, 90, seed=3), meshgen.QUAD4)])
def test_reduces_to_fixed_types(make, et):
    conn, N = make()
    off, idx = meshgen.poly_from_conn(conn)
    for pf, ff in ((oracle.poly_node_csr, oracle.node_csr), (oracle.poly_elem_csr, oracle.elem_csr),
                   (oracle.poly_shared_csr, oracle.node_shared_csr)):
        a, b = pf(off, idx, N), ff(et, conn, N)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("seed,M,N,kmin,kmax", [(1, 40, 30, 3, 7), (2, 200, 60, 3, 12), (3, 15, 200, 3, 5),
                                               (4, 60, 12, 3, 12)])
def test_brute_force(seed, M, N, kmin, kmax):
    off, idx, N = meshgen.random_poly(M, N, kmin, kmax, seed)
    for mode, fn in (("node", oracle.poly_node_csr), ("elem", oracle.poly_elem_csr),
                     ("shared", oracle.poly_shared_csr)):
        got = _lists(*fn(off, idx, N))
        assert got == _brute(off, idx, N, mode), mode


@pytest.mark.parametrize("r,c,seed", [(1, 1, 0), (5, 7, 1604), (16, 9, 7)])
def test_mixed_grid_closed_form(r, c, seed):
    off, idx, N = meshgen.poly_mixed_grid(r, c, seed)
    split = int((off.numel() - 1) - r * c)          # every split cell adds one element and one edge
    o, i = oracle.poly_node_csr(off, idx, N)
    assert len(i) == 2 * (r * (c + 1) + c * (r + 1) + split)
    # corner node 0 always has its two grid neighbours, plus the diagonal when cell 0 is split 00-11
    assert set(i[o[0]:o[1]].tolist()) >= {1, c + 1}


@pytest.mark.parametrize("r,c", [(1, 1), (4, 6), (9, 5)])
def test_honeycomb_euler_and_valence(r, c):
    off, idx, N = meshgen.honeycomb(r, c)
    o, i = oracle.poly_node_csr(off, idx, N)
    deg = np.diff(o)
    used = int((deg > 0).sum())
    E = len(i) // 2
    assert used - E + r * c == 1                        # a disk
    assert set(np.unique(deg)) <= {0, 2, 3} and (deg.max() == 3) == (r * c > 1)
    # every hexagon's 6 ring neighbours, in the node lists
    idn = idx.numpy()
    for e in range(r * c):
        ring = idn[6 * e:6 * e + 6]
        for p in range(6):
            assert ring[(p + 1) % 6] in i[o[ring[p]]:o[ring[p] + 1]]


@pytest.mark.parametrize("make", [lambda: meshgen.poly_mixed_grid(6, 5, 11), lambda: meshgen.honeycomb(3, 4),
                                  lambda: meshgen.random_poly(80, 40, 3, 9, 5)])
def test_shared_is_incidence_pattern(make):
    off, idx, N = make()
    off, idx = off.numpy(), idx.numpy()
    M = len(off) - 1
    B = np.zeros((M, N), dtype=np.int64)
    for e in range(M):
        B[e, idx[off[e]:off[e + 1]]] = 1
    P = (B.T @ B) > 0
    np.fill_diagonal(P, False)
    o, i = oracle.poly_shared_csr(off, idx, N)
    for v in range(N):
        assert i[o[v]:o[v + 1]].tolist() == np.nonzero(P[v])[0].tolist()


def test_relabel_equivariance():
    off, idx, N = meshgen.poly_mixed_grid(7, 6, 3)
    o1, i1 = oracle.poly_node_csr(off, idx, N)
    off2, idx2 = meshgen.poly_relabel(off, idx, N, 17, 23)
    o2, i2 = oracle.poly_node_csr(off2, idx2, N)
    pi = meshgen.seeded_permutation(N, 17)
    for v in range(N):
        assert sorted(pi[i1[o1[v]:o1[v + 1]]].tolist()) == i2[o2[pi[v]]:o2[pi[v] + 1]].tolist()


def test_validation_rules():
    P = lambda rings: (np.cumsum([0] + [len(r) for r in rings]), np.concatenate([np.array(r) for r in rings]))
    # SPEC validate_mesh examples as polygons
    assert oracle.poly_validate(*P([[0, 1, 2]]), 3) == (oracle.OK, -1, -1)
    assert oracle.poly_validate(*P([[0, 1, 3]]), 3) == (oracle.ERR_RANGE, 0, 2)
    assert oracle.poly_validate(*P([[0, 1, 1]]), 3)[:2] == (oracle.ERR_DEGENERATE, 0)
    # R18: arity before range within an element; the lowest element decides
    assert oracle.poly_validate(*P([[0, 1, 2], [5, 9], [0, 9, 9]]), 4) == (oracle.ERR_ARITY, 1, -1)
    assert oracle.poly_validate(*P([[0, 1, 2, 3], [0, 9, 9], [7, 8]]), 4) == (oracle.ERR_RANGE, 1, 1)
    assert oracle.poly_validate(*P([[0, 1, 2, 3, 2, 9]]), 10) == (oracle.ERR_DEGENERATE, 0, 4)
    with pytest.raises(oracle.OracleMeshError) as ei:
        oracle.poly_node_csr(*P([[0, 1, 2], [3, 4]]), 5)
    assert (ei.value.code, ei.value.elem, ei.value.pos) == (oracle.ERR_ARITY, 1, -1)
    # empty mesh, isolated nodes
    o, i = oracle.poly_node_csr(np.zeros(1, np.int64), np.zeros(0, np.int32), 4)
    assert o.tolist() == [0, 0, 0, 0, 0] and len(i) == 0


@pytest.mark.parametrize("make", [lambda: meshgen.random_poly(200, 60, 3, 12, 2), lambda: meshgen.poly_mixed_grid(9, 7, 5),
                                  lambda: meshgen.honeycomb(5, 4)])
def test_sampled_form_matches_full(make):
    from oracle import stages
    off, idx, N = make()
    smp = stages.poly_neighbors_sample(off, idx, N, list(range(0, N, 3)))
    o, i = oracle.poly_node_csr(off, idx, N)
    eo, ei = oracle.poly_elem_csr(off, idx, N)
    so, si = oracle.poly_shared_csr(off, idx, N)
    for v, (a, b, c) in smp.items():
        assert a.tolist() == i[o[v]:o[v + 1]].tolist()
        assert b.tolist() == ei[eo[v]:eo[v + 1]].tolist()
        assert c.tolist() == si[so[v]:so[v + 1]].tolist()


@pytest.mark.parametrize("seed,M,N,kmin,kmax", [(1, 40, 30, 3, 7), (2, 200, 60, 3, 12), (4, 60, 12, 3, 12)])
def test_range_mode_brute_force(seed, M, N, kmin, kmax):
    """Node-range mode == brute-force rows lo..hi-1 for every mode, every range end."""
    off, idx, N = meshgen.random_poly(M, N, kmin, kmax, seed)
    exp = {oracle.NODE: _brute(off, idx, N, "node"), oracle.ELEM: _brute(off, idx, N, "elem"),
           oracle.SHARED: _brute(off, idx, N, "shared")}
    for lo in range(0, N + 1, 3):
        for hi in (lo, min(N, lo + 1), min(N, lo + 7), N):
            for mode, rows in exp.items():
                o, i = oracle.poly_csr_range(mode, off, idx, N, lo, hi)
                assert o[0] == 0 and _lists(o, i) == [list(r) for r in rows[lo:hi]], (mode, lo, hi)
