"""Step-by-step oracle of the paper's GPU pipeline — TEST INFRASTRUCTURE ONLY.

Each function is one step of PAPER.md §2.2.1 ("The Finding of Neighboring Nodes", L218-248) or
§2.2.2 (L250-264), written plainly in numpy in the paper's order and notation.  Library
primitives (np.lexsort, np.argsort, np.cumsum) serve as steps; nothing is blocked, fused or
reordered.  Paper-silent points follow DESIGN.md §"Readings" (R1..R14); each function names the
ones it uses.  Parity pins are in tests/test_oracle_*.py (listed in DESIGN.md §"Oracle pins").
"""
from __future__ import annotations

import numpy as np

TRI3, QUAD4, TET4, HEX8 = 0, 1, 2, 3

# Element edge tables (§2.1.1 "connected using an edge"; triangles spelled out
# in §2.2.1; other types per reading R4).  The order of edges fixes the order pairs are
# created in (reading R5: element-major, edge order below, forward pair then reverse pair).
EDGES = {
    TRI3: ((0, 1), (1, 2), (2, 0)),
    QUAD4: ((0, 1), (1, 2), (2, 3), (3, 0)),
    TET4: ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)),
    HEX8: ((0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
           (0, 4), (1, 5), (2, 6), (3, 7)),
}
ARITY = {TRI3: 3, QUAD4: 4, TET4: 4, HEX8: 8}


def _conn(conn):
    if hasattr(conn, "detach"):
        conn = conn.detach().cpu().numpy()
    conn = np.asarray(conn)
    # int32 ids are kept as they are (a config-5 connectivity is 3.15 GB); widened otherwise
    return conn if conn.dtype in (np.int32, np.int64) else conn.astype(np.int64)


# ---- step 1: pair creation ------------------------------------------------------------------
def expand_node_pairs(etype: int, conn):
    """PAPER.md §2.2.1: "we can form three edges (pairs of integers) for a triangle when
    the three nodes ... are organized in CCW order and another three pairs when ... CW ... a
    triangle can produce six pairs of integers."  Generalised per R4: every element edge (i, j)
    yields (conn[i], conn[j]) then (conn[j], conn[i]).  Returns the paper's "two arrays of
    integers" (Fig. 1d): keys (first node) and values (second node), element-major (R5)."""
    c = _conn(conn).reshape(-1, ARITY[etype])
    keys, vals = [], []
    for (i, j) in EDGES[etype]:
        keys.append(np.stack([c[:, i], c[:, j]], 1))
        vals.append(np.stack([c[:, j], c[:, i]], 1))
    keys = np.stack(keys, 1).reshape(-1)      # [M, nedges, 2] -> slot e*2E + 2*edge + dir
    vals = np.stack(vals, 1).reshape(-1)
    return keys, vals


def expand_elem_pairs(etype: int, conn):
    """PAPER.md §2.1.2 L157-161 / §2.2.2: "the first integer value of any pair is the
    index of a node in an element; and the second value ... is the index of the element itself".
    Element-major, local node order (R5)."""
    c = _conn(conn).reshape(-1, ARITY[etype])
    M, k = c.shape
    keys = c.reshape(-1)
    vals = np.repeat(np.arange(M, dtype=np.int64), k)
    return keys, vals


# ---- step 2: sort -------------------------------------------------------------------------------
def sort_pairs(keys, vals):
    """PAPER.md §2.2.1: "sort those pairs according to the first array of integers"
    (thrust::sort_by_key).  Reading R2: within one key the values come out ascending (a
    lexicographic sort on (key, value)), which makes the output canonical."""
    order = np.lexsort((vals, keys))
    return keys[order], vals[order]


def stable_sort_by_key(keys, vals):
    """Element mode (§2.2.2, "sort according to the first array of integers"), reading
    R3: a stable sort by key; element-major creation order then leaves each node's elements
    ascending."""
    order = np.argsort(keys, kind="stable")
    return keys[order], vals[order]


# ---- dedupe (paper silent; reading R1) ---------------------------------------------------------
def unique_pairs(keys, vals):
    """Reading R1 (north_star: "deduplicates by adjacent difference"): after the sort, drop every
    pair equal to its predecessor."""
    if keys.size == 0:
        return keys, vals
    keep = np.ones(keys.size, dtype=bool)
    keep[1:] = (keys[1:] != keys[:-1]) | (vals[1:] != vals[:-1])
    return keys[keep], vals[keep]


# ---- step 3: segmented reduction and scan ----------------------------------------------------
def reduce_by_key_ones(sorted_keys):
    """PAPER.md §2.2.1: "create a helper array containing the same value 1 ... then
    perform a parallel segmented reduction" (thrust::reduce_by_key) -> (unique keys, counts)."""
    ones = np.ones(sorted_keys.size, dtype=np.int64)
    if sorted_keys.size == 0:
        return sorted_keys[:0], ones[:0]
    start = np.ones(sorted_keys.size, dtype=bool)
    start[1:] = sorted_keys[1:] != sorted_keys[:-1]
    seg = np.cumsum(start) - 1
    counts = np.zeros(int(seg[-1]) + 1, dtype=np.int64)
    np.add.at(counts, seg, ones)
    return sorted_keys[start], counts


def first_positions_by_key(sorted_keys):
    """PAPER.md §2.2.1: "create a helper array of sequenced integers ... then perform a
    parallel segmented scan by using thrust::unique_by_keys()" -> (unique keys, first index)
    (reading R12)."""
    seq = np.arange(sorted_keys.size, dtype=np.int64)
    if sorted_keys.size == 0:
        return sorted_keys[:0], seq[:0]
    start = np.ones(sorted_keys.size, dtype=bool)
    start[1:] = sorted_keys[1:] != sorted_keys[:-1]
    return sorted_keys[start], seq[start]


def exclusive_scan(counts):
    """offsets[0] = 0, offsets[i+1] = offsets[i] + counts[i] (the "first indices" of L487-489)."""
    out = np.zeros(len(counts) + 1, dtype=np.int64)
    out[1:] = np.cumsum(np.asarray(counts, dtype=np.int64))
    return out


def dense_counts(unique_keys, counts, num_nodes):
    """Per-vertex "numbers" (L487-489) for all num_nodes vertices; unused vertices get 0 (R7)."""
    out = np.zeros(num_nodes, dtype=np.int64)
    out[np.asarray(unique_keys, dtype=np.int64)] = counts
    return out


# ---- whole pipeline, step by step ----------------------------------------------------------------
def node_csr(etype: int, conn, num_nodes: int):
    keys, vals = expand_node_pairs(etype, conn)
    keys, vals = sort_pairs(keys, vals)
    keys, vals = unique_pairs(keys, vals)
    uk, cnt = reduce_by_key_ones(keys)
    offsets = exclusive_scan(dense_counts(uk, cnt, num_nodes))
    return offsets, vals.astype(np.int32)


def elem_csr(etype: int, conn, num_nodes: int):
    keys, vals = expand_elem_pairs(etype, conn)
    keys, vals = stable_sort_by_key(keys, vals)
    uk, cnt = reduce_by_key_ones(keys)
    offsets = exclusive_scan(dense_counts(uk, cnt, num_nodes))
    return offsets, vals.astype(np.int32)


# ---- one-vertex-at-a-time forms (full-size sampled parity) --------------------------------------
def node_neighbors_sample(etype: int, conn, num_nodes: int, sample):
    """adj(v) for each v in ``sample`` straight from the definition (PAPER.md: "any pair
    of nodes connected by an edge is the one-ring neighboring node for each other"): scan every
    element containing v, collect the other end of each of its edges at v.  -> {v: sorted array}"""
    c = _conn(conn).reshape(-1, ARITY[etype])
    sample = np.asarray(sample, dtype=np.int64)
    lut = np.zeros(num_nodes, dtype=bool)
    lut[sample] = True
    rows = np.nonzero(lut[c].any(1))[0]
    sub = c[rows]
    out = {int(v): set() for v in sample}
    for (i, j) in EDGES[etype]:
        a, b = sub[:, i], sub[:, j]
        for x, y in zip(a.tolist(), b.tolist()):
            if x in out:
                out[x].add(y)
            if y in out:
                out[y].add(x)
    return {v: np.array(sorted(s), dtype=np.int32) for v, s in out.items()}


def elem_neighbors_sample(etype: int, conn, num_nodes: int, sample):
    """inc(v) for each v in ``sample`` ("any element is directly the one-ring
    neighboring element for those nodes it contains")."""
    c = _conn(conn).reshape(-1, ARITY[etype])
    sample = np.asarray(sample, dtype=np.int64)
    lut = np.zeros(num_nodes, dtype=bool)
    lut[sample] = True
    rows = np.nonzero(lut[c].any(1))[0]
    sub = c[rows]
    out = {}
    for v in sample.tolist():
        out[v] = rows[(sub == v).any(1)].astype(np.int32)
    return out


def poly_neighbors_sample(off, idx, num_nodes: int, sample):
    """Polygon meshes (ring e = idx[off[e]:off[e+1]]), for each v in ``sample`` straight from the
    definitions: the elements whose ring contains v (ascending), v's two ring neighbours in each
    of them (ring-edge adjacency), and all other nodes of them (element-sharing adjacency).
    -> {v: (node sorted array, elem array, shared sorted array)}"""
    off = np.asarray(off.cpu() if hasattr(off, "cpu") else off, dtype=np.int64)
    idx = np.asarray(idx.cpu() if hasattr(idx, "cpu") else idx, dtype=np.int64)
    sample = np.asarray(sample, dtype=np.int64)
    lut = np.zeros(num_nodes, dtype=bool)
    lut[sample] = True
    pos = np.nonzero(lut[idx])[0]                              # ring entries holding a sampled node
    elem = np.searchsorted(off, pos, side="right") - 1         # their elements
    out = {int(v): (set(), [], set()) for v in sample}
    for p, e in zip(pos.tolist(), elem.tolist()):
        b, k = int(off[e]), int(off[e + 1] - off[e])
        ring = idx[b:b + k].tolist()
        q = p - b
        v = ring[q]
        node, inc, shared = out[v]
        node.add(ring[(q - 1) % k])
        node.add(ring[(q + 1) % k])
        inc.append(e)
        shared.update(x for x in ring if x != v)
    return {v: (np.array(sorted(a), dtype=np.int32), np.array(b, dtype=np.int32),
                np.array(sorted(c), dtype=np.int32)) for v, (a, b, c) in out.items()}
