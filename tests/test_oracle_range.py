"""Pins for the oracle's node-range / T-thread mode and the one-vertex sampled forms, CPU only.

SURVEY §8(c): "an optional T-thread mode where thread t owns node range t and scans all elements;
the output is identical".  These forms are what the full-size GPU parity tests (configs 3-5) and
bench.py's parity gate compare against, so each is pinned to something other than itself:
brute force from the definitions on tiny meshes, the closed-form CSRs of the
structured generators (Kuhn / hex / tri grid), and the pinned one-thread oracle on the SMALL
corpus.  A wrong range bound, a dropped boundary vertex, a slice stitched at the wrong offset or a
per-thread set that misses pairs from elements outside its range each fail one of them.
"""
import numpy as np
import pytest

import meshgen
import oracle
from oracle import stages
from test_oracle_pins import (TINY, TINY_TYPES, _hex_closed_form, _kuhn_closed_form, _grid_closed_form_tri,
                              _slices, brute_elem, brute_node)

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")

SMALL = [
    ("kuhn_7", meshgen.TET4, lambda: meshgen.kuhn_tets(7)),
    ("hex_6_relabelled", meshgen.HEX8, lambda: (meshgen.relabel(*meshgen.hex_grid(6), 1604, 4689), 7 ** 3)),
    ("sphere_40x21", meshgen.TRI3, lambda: meshgen.uv_sphere(40, 21)),
    ("quad_9x13", meshgen.QUAD4, lambda: meshgen.quad_grid(9, 13)),
    ("rand_tet", meshgen.TET4, lambda: meshgen.random_mesh(meshgen.TET4, 3000, 700, seed=11)),
    ("rand_hex_sparse", meshgen.HEX8, lambda: meshgen.random_mesh(meshgen.HEX8, 50, 2000, seed=12)),
    ("fan_40", meshgen.TRI3, lambda: meshgen.nonmanifold_fan(40)),
]

FULL = {oracle.NODE: oracle.node_csr, oracle.ELEM: oracle.elem_csr, oracle.SHARED: oracle.node_shared_csr}


def _conn_n(made):
    conn, N = made[0], made[1]
    return conn, N


@pytest.mark.parametrize("name,make", TINY)
@pytest.mark.parametrize("T", [1, 2, 3, 5, 1000])
def test_mt_brute_force(name, make, T):
    """T-thread CSR == brute force from the definitions (edge relation derived without the
    oracle's tables), for T dividing N unevenly and T > N."""
    conn, N = make()
    et = TINY_TYPES[name]
    o, i, used = oracle.csr_mt(oracle.NODE, et, conn, N, T)
    assert used == max(1, min(T, N))
    assert _slices(o, i) == brute_node(et, conn, N), name
    o, i, _ = oracle.csr_mt(oracle.ELEM, et, conn, N, T)
    assert _slices(o, i) == brute_elem(et, conn, N), name


@pytest.mark.parametrize("name,make", TINY)
def test_range_brute_force(name, make):
    """Every [lo, hi) slice (including empty ones and the two ends) == brute force rows lo..hi-1."""
    conn, N = make()
    et = TINY_TYPES[name]
    bn, be = brute_node(et, conn, N), brute_elem(et, conn, N)
    for lo in range(N + 1):
        for hi in (lo, min(N, lo + 1), min(N, lo + 3), N):
            o, i = oracle.csr_range(oracle.NODE, et, conn, N, lo, hi)
            assert o[0] == 0 and len(o) == hi - lo + 1
            assert _slices(o, i) == bn[lo:hi]
            o, i = oracle.csr_range(oracle.ELEM, et, conn, N, lo, hi)
            assert _slices(o, i) == be[lo:hi]


@pytest.mark.parametrize("n", [3, 5])
def test_mt_closed_form_kuhn(n):
    conn, N = meshgen.kuhn_tets(n)
    adj, inc = _kuhn_closed_form(n)
    for T in (1, 4, 7, N):
        o, i, _ = oracle.csr_mt(oracle.NODE, meshgen.TET4, conn, N, T)
        assert _slices(o, i) == adj
        o, i, _ = oracle.csr_mt(oracle.ELEM, meshgen.TET4, conn, N, T)
        assert _slices(o, i) == inc
    lo, hi = N // 3, N // 3 + 17
    assert _slices(*oracle.csr_range(oracle.NODE, meshgen.TET4, conn, N, lo, hi)) == adj[lo:hi]
    assert _slices(*oracle.csr_range(oracle.ELEM, meshgen.TET4, conn, N, lo, hi)) == inc[lo:hi]


def test_mt_closed_form_hex_and_tri():
    conn, N = meshgen.hex_grid(4)
    adj, inc = _hex_closed_form(4)
    o, i, _ = oracle.csr_mt(oracle.NODE, meshgen.HEX8, conn, N, 6)
    assert _slices(o, i) == adj
    o, i, _ = oracle.csr_mt(oracle.ELEM, meshgen.HEX8, conn, N, 6)
    assert _slices(o, i) == inc
    conn, N = meshgen.tri_grid(7, 9)
    adj, inc = _grid_closed_form_tri(7, 9)
    o, i, _ = oracle.csr_mt(oracle.NODE, meshgen.TRI3, conn, N, 9)
    assert _slices(o, i) == adj
    o, i, _ = oracle.csr_mt(oracle.ELEM, meshgen.TRI3, conn, N, 9)
    assert _slices(o, i) == inc


@pytest.mark.parametrize("name,et,make", SMALL)
def test_mt_equals_one_thread_small(name, et, make):
    """On the SMALL corpus (non-manifold fans, isolated vertices, relabelled hex, poles) the
    T-thread and range forms equal the pinned one-thread oracle, for all three modes."""
    conn, N = _conn_n(make())
    for mode, fn in FULL.items():
        ro, ri = fn(et, conn, N)
        for T in (2, 3, 8, 33):
            o, i, _ = oracle.csr_mt(mode, et, conn, N, T)
            assert np.array_equal(o, ro) and np.array_equal(i, ri), (name, mode, T)
        lo, hi = N // 5, N // 5 + N // 7
        o, i = oracle.csr_range(mode, et, conn, N, lo, hi)
        assert np.array_equal(o, ro[lo:hi + 1] - ro[lo]), (name, mode)
        assert np.array_equal(i, ri[ro[lo]:ro[hi]]), (name, mode)


def test_mt_validation_and_empty():
    """Validation is global and precedes every range: the lowest offending element is reported,
    whatever range a thread owns; empty meshes give all-zero offsets."""
    conn, N = meshgen.kuhn_tets(3)
    bad = conn.clone()
    bad[40, 2] = N                      # out of range
    bad[7, 3] = bad[7, 1]               # repeated node, lower element
    with pytest.raises(oracle.OracleMeshError) as ex:
        oracle.csr_mt(oracle.NODE, meshgen.TET4, bad, N, 4)
    assert (ex.value.code, ex.value.elem, ex.value.pos) == (oracle.ERR_DEGENERATE, 7, 3)
    with pytest.raises(oracle.OracleMeshError) as ex:
        oracle.csr_range(oracle.ELEM, meshgen.TET4, bad, N, N - 2, N)
    assert (ex.value.code, ex.value.elem) == (oracle.ERR_DEGENERATE, 7)
    import torch
    empty = torch.zeros((0, 4), dtype=torch.int32)
    o, i, _ = oracle.csr_mt(oracle.NODE, meshgen.TET4, empty, 5, 3)
    assert o.tolist() == [0] * 6 and i.size == 0
    o, i, _ = oracle.csr_mt(oracle.ELEM, meshgen.TET4, empty, 0, 3)
    assert o.tolist() == [0] and i.size == 0


# ---- the one-vertex sampled forms (stages.node_neighbors_sample / elem_neighbors_sample) ------
@pytest.mark.parametrize("name,make", TINY)
def test_sampled_forms_brute_force(name, make):
    conn, N = make()
    et = TINY_TYPES[name]
    bn, be = brute_node(et, conn, N), brute_elem(et, conn, N)
    sample = list(range(N))
    sn = stages.node_neighbors_sample(et, conn, N, sample)
    se = stages.elem_neighbors_sample(et, conn, N, sample)
    for v in sample:
        assert sn[v].tolist() == bn[v], (name, v)
        assert se[v].tolist() == be[v], (name, v)


def test_sampled_forms_closed_form_kuhn():
    n = 5
    conn, N = meshgen.kuhn_tets(n)
    adj, inc = _kuhn_closed_form(n)
    sample = [0, 1, n, N // 2, N - 1, 37, 100]
    sn = stages.node_neighbors_sample(meshgen.TET4, conn, N, sample)
    se = stages.elem_neighbors_sample(meshgen.TET4, conn, N, sample)
    for v in sample:
        assert sn[v].tolist() == adj[v] and se[v].tolist() == inc[v], v


@pytest.mark.parametrize("name,et,make", SMALL)
def test_sampled_forms_equal_full_oracle(name, et, make):
    conn, N = _conn_n(make())
    ro, ri = oracle.node_csr(et, conn, N)
    eo, ei = oracle.elem_csr(et, conn, N)
    rng = np.random.default_rng(5)
    sample = sorted(set(rng.integers(0, N, 40).tolist()) | {0, N - 1})
    sn = stages.node_neighbors_sample(et, conn, N, sample)
    se = stages.elem_neighbors_sample(et, conn, N, sample)
    for v in sample:
        assert np.array_equal(sn[v], ri[ro[v]:ro[v + 1]]), (name, v)
        assert np.array_equal(se[v], ei[eo[v]:eo[v + 1]]), (name, v)
