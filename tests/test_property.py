"""Property-based tests (hypothesis): random meshes of every element type, random sizes, node counts
with isolated vertices, and random corruptions.

CPU: the oracle against brute force from the definitions — another pin, over a
much wider input space than the fixed corpus.
GPU: the CUDA path through the C ABI against the oracle, bit for bit, on every element path and the
one-CTA small path, including the validation error (lowest element, range before repeated node)."""
import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import meshgen
import oracle
from test_oracle_pins import _slices, brute_elem, brute_node

TYPES = [meshgen.TRI3, meshgen.QUAD4, meshgen.TET4, meshgen.HEX8]


@st.composite
def meshes(draw, max_elems=40, max_nodes=30):
    """Random element type, sizes and seed; the rows (k distinct nodes each, non-manifold edges and
    isolated vertices included) come from meshgen.random_mesh with that seed."""
    et = draw(st.sampled_from(TYPES))
    k = meshgen.ARITY[et]
    N = draw(st.integers(min_value=k, max_value=max_nodes))
    M = draw(st.integers(min_value=0, max_value=max_elems))
    seed = draw(st.integers(min_value=0, max_value=2 ** 31 - 1))
    conn, _ = meshgen.random_mesh(et, M, N, seed=seed)
    return et, conn.reshape(M, k).contiguous(), N


@st.composite
def corrupted(draw):
    et, conn, N = draw(meshes(max_elems=30, max_nodes=20))
    M, k = conn.shape
    if M == 0:
        return et, conn, N
    for _ in range(draw(st.integers(min_value=1, max_value=3))):
        e = draw(st.integers(min_value=0, max_value=M - 1))
        p = draw(st.integers(min_value=0, max_value=k - 1))
        kind = draw(st.sampled_from(["range_hi", "range_lo", "dup"]))
        if kind == "range_hi":
            conn[e, p] = N + draw(st.integers(min_value=0, max_value=5))
        elif kind == "range_lo":
            conn[e, p] = -1 - draw(st.integers(min_value=0, max_value=5))
        else:
            q = draw(st.integers(min_value=0, max_value=k - 1))
            if q != p:
                conn[e, p] = conn[e, q]
    return et, conn, N


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(meshes(max_elems=12, max_nodes=12))
def test_oracle_equals_brute_force(m):
    et, conn, N = m
    assert _slices(*oracle.node_csr(et, conn, N)) == brute_node(et, conn, N)
    assert _slices(*oracle.elem_csr(et, conn, N)) == brute_elem(et, conn, N)
    o, i, _ = oracle.csr_mt(oracle.NODE, et, conn, N, 3)
    assert _slices(o, i) == brute_node(et, conn, N)


@settings(max_examples=60, deadline=None)
@given(corrupted())
def test_oracle_validation_order(m):
    """The oracle's validation = the lowest element, range before repeated node, lowest position —
    recomputed here by a direct scan (reading R8)."""
    et, conn, N = m
    c = conn.numpy()
    exp = (oracle.OK, -1, -1)
    for e in range(c.shape[0]):
        row = c[e].tolist()
        bad = [p for p, v in enumerate(row) if v < 0 or v >= N]
        if bad:
            exp = (oracle.ERR_RANGE, e, bad[0])
            break
        dup = [p for p in range(1, len(row)) if row[p] in row[:p]]
        if dup:
            exp = (oracle.ERR_DEGENERATE, e, dup[0])
            break
    assert oracle.validate(et, conn, N) == exp


# ---------------------------------------------------------------------------------------------
# GPU: the CUDA path against the oracle
# ---------------------------------------------------------------------------------------------
def _mn():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1604_04689_b200 as mn
    return mn


@pytest.mark.gpu
@settings(max_examples=80, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(meshes(max_elems=300, max_nodes=200), st.sampled_from(["auto", "radix", "transpose", "msd"]))
def test_gpu_equals_oracle_random(m, path):
    mn = _mn()
    et, conn, N = m
    mn.set_elem_path(path)
    try:
        (no, ni), (eo, ei) = mn.find_neighbors(conn.cuda(), et, N)
    finally:
        mn.set_elem_path("auto")
    ro, ri = oracle.node_csr(et, conn, N)
    so, si = oracle.elem_csr(et, conn, N)
    assert np.array_equal(no.cpu().numpy(), ro) and np.array_equal(ni.cpu().numpy(), ri)
    assert np.array_equal(eo.cpu().numpy(), so) and np.array_equal(ei.cpu().numpy(), si)


@pytest.mark.gpu
@settings(max_examples=60, deadline=None)
@given(corrupted(), st.sampled_from(["auto", "radix", "transpose"]))
def test_gpu_validation_random(m, path):
    mn = _mn()
    et, conn, N = m
    code, e, p = oracle.validate(et, conn, N)
    mn.set_elem_path(path)
    try:
        if code == oracle.OK:
            mn.find_neighbors(conn.cuda(), et, N)
            return
        with pytest.raises(mn.MeshError) as ex:
            mn.find_neighbors(conn.cuda(), et, N)
    finally:
        mn.set_elem_path("auto")
    want = {oracle.ERR_RANGE: mn.MN_ERR_INDEX_OUT_OF_RANGE, oracle.ERR_DEGENERATE: mn.MN_ERR_DEGENERATE}[code]
    assert (ex.value.code, ex.value.elem, ex.value.pos) == (want, e, p)
