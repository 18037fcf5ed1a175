"""Seeded synthetic mesh generators — the ONLY module shared by the oracle side and the CUDA side.

It builds connectivity arrays (``int32 [M, k]`` row-major, 0-based) and nothing else: no pair
expansion, no sorting, no adjacency — none of the method's arithmetic (§2.2) lives here.
Shapes follow the paper's workloads (closed triangle surfaces with F ≈ 2V, Table 1,
L313-406) and BASELINE.json's five configs; the exact recipes are in DESIGN.md §"Input recipe".

Everything is written with torch integer ops so the same function yields bit-identical arrays on
CPU (tests, oracle) and on CUDA (bench: inputs generated straight into HBM).  Permutations use a
splitmix64 hash ranked by argsort (numpy uint64 arithmetic), seeded; they are bijections, so the
ranking is unique.
"""
from __future__ import annotations

import numpy as np
import torch

# element-type codes, same numbering as include/meshnbr.h (mn_elem_type)
TRI3, QUAD4, TET4, HEX8 = 0, 1, 2, 3
ARITY = {TRI3: 3, QUAD4: 4, TET4: 4, HEX8: 8}
TYPE_NAMES = {TRI3: "tri3", QUAD4: "quad4", TET4: "tet4", HEX8: "hex8"}


def _dev(device):
    return torch.device(device) if device is not None else torch.device("cpu")


# --------------------------------------------------------------------------------------------
# structured generators
# --------------------------------------------------------------------------------------------
def tri_grid(rows: int, cols: int, device=None):
    """Freudenthal triangle grid: (cols+1) x (rows+1) nodes, node (i, j) -> i + (cols+1) j.

    Cell (i, j) (i < cols, j < rows) -> triangles (v00, v10, v11), (v00, v11, v01), element ids
    2 (i + cols j) + {0, 1}.  Same-diagonal split as SPEC.md generate_grid."""
    d = _dev(device)
    i = torch.arange(cols, device=d, dtype=torch.int64)
    j = torch.arange(rows, device=d, dtype=torch.int64)
    jj, ii = torch.meshgrid(j, i, indexing="ij")          # row-major over (j, i)
    w = cols + 1
    v00 = ii + w * jj
    v10 = v00 + 1
    v01 = v00 + w
    v11 = v01 + 1
    t0 = torch.stack([v00, v10, v11], -1)
    t1 = torch.stack([v00, v11, v01], -1)
    conn = torch.stack([t0, t1], -2).reshape(-1, 3)
    return conn.to(torch.int32).contiguous(), (rows + 1) * (cols + 1)


def quad_grid(rows: int, cols: int, device=None):
    """Quad grid, same node numbering as tri_grid; cell (i, j) -> (v00, v10, v11, v01)."""
    d = _dev(device)
    i = torch.arange(cols, device=d, dtype=torch.int64)
    j = torch.arange(rows, device=d, dtype=torch.int64)
    jj, ii = torch.meshgrid(j, i, indexing="ij")
    w = cols + 1
    v00 = ii + w * jj
    conn = torch.stack([v00, v00 + 1, v00 + 1 + w, v00 + w], -1).reshape(-1, 4)
    return conn.to(torch.int32).contiguous(), (rows + 1) * (cols + 1)


def uv_sphere(nlon: int, nrings: int, device=None):
    """Closed genus-0 triangulated sphere: north pole 0, ring r in [0, nrings), longitude l in
    [0, nlon): id 1 + nlon r + l, south pole 1 + nlon nrings.

    Top fan (0, rv(0,l), rv(0,l+1)); bands (a,b,c), (a,c,d) with a=rv(r,l), b=rv(r+1,l),
    c=rv(r+1,l+1), d=rv(r,l+1); bottom fan (S, rv(R-1,l+1), rv(R-1,l)).
    M = 2 nlon nrings, N = nlon nrings + 2."""
    d = _dev(device)
    L, R = nlon, nrings
    l = torch.arange(L, device=d, dtype=torch.int64)
    lp = (l + 1) % L

    def rv(r, ll):
        return 1 + L * r + ll

    south = 1 + L * R
    top = torch.stack([torch.zeros_like(l), rv(0, l), rv(0, lp)], -1)
    parts = [top]
    if R > 1:
        r = torch.arange(R - 1, device=d, dtype=torch.int64)[:, None]
        a, b, c, dd = rv(r, l), rv(r + 1, l), rv(r + 1, lp), rv(r, lp)
        band = torch.stack([torch.stack([a, b, c], -1), torch.stack([a, c, dd], -1)], -2)
        parts.append(band.reshape(-1, 3))
    bot = torch.stack([torch.full_like(l, south), rv(R - 1, lp), rv(R - 1, l)], -1)
    parts.append(bot)
    conn = torch.cat(parts, 0)
    return conn.to(torch.int32).contiguous(), L * R + 2


# the 6 axis permutations in lexicographic order (Kuhn / Freudenthal simplices of a cube)
KUHN_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def kuhn_tets(n: int, device=None, cell_begin: int = 0, cell_end: int | None = None):
    """Kuhn-subdivided n^3 cube: node (i,j,k) -> i + (n+1)(j + (n+1)k); cell c = ci + n(cj + n ck);
    tet 6c + p (p indexes KUHN_PERMS) = (x, x+e_p0, x+e_p0+e_p1, x+(1,1,1)).

    ``cell_begin/cell_end`` select a contiguous cell range (elements 6*cell_begin .. 6*cell_end),
    which is exactly an element shard of the full mesh (used by the multi-GPU path)."""
    d = _dev(device)
    ncell = n * n * n
    cell_end = ncell if cell_end is None else cell_end
    c = torch.arange(cell_begin, cell_end, device=d, dtype=torch.int64)
    ci = c % n
    cj = (c // n) % n
    ck = c // (n * n)
    w = n + 1
    base = ci + w * (cj + w * ck)
    step = (1, w, w * w)
    tets = []
    for p in KUHN_PERMS:
        a = base
        b = a + step[p[0]]
        cc = b + step[p[1]]
        dd = base + 1 + w + w * w
        tets.append(torch.stack([a, b, cc, dd], -1))
    conn = torch.stack(tets, 1).reshape(-1, 4)
    return conn.to(torch.int32).contiguous(), w * w * w


def hex_grid(n: int, device=None):
    """n^3 hexahedra in VTK_HEXAHEDRON local order: 0-3 bottom ring (z=k), 4-7 top ring, 4 above 0.
    Node (i,j,k) -> i + (n+1)(j + (n+1)k); element id ci + n(cj + n ck)."""
    d = _dev(device)
    c = torch.arange(n * n * n, device=d, dtype=torch.int64)
    ci = c % n
    cj = (c // n) % n
    ck = c // (n * n)
    w = n + 1
    b = ci + w * (cj + w * ck)
    ring = [b, b + 1, b + 1 + w, b + w]
    top = [x + w * w for x in ring]
    conn = torch.stack(ring + top, -1)
    return conn.to(torch.int32).contiguous(), w * w * w


# --------------------------------------------------------------------------------------------
# seeded permutations (splitmix64 ranks)
# --------------------------------------------------------------------------------------------
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """The first ``count`` outputs of splitmix64 seeded with ``seed`` (Steele et al. 2014)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.arange(1, count + 1, dtype=np.uint64) * _GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def seeded_permutation(count: int, seed: int) -> np.ndarray:
    """A uniformly scrambled permutation of range(count): the rank order of splitmix64 outputs.
    splitmix64's finaliser is a bijection of its 64-bit state, so all keys are distinct and the
    permutation is unique (no tie-breaking)."""
    return np.argsort(splitmix64(seed, count), kind="stable").astype(np.int64)


def relabel(conn: torch.Tensor, num_nodes: int, node_seed: int | None, elem_seed: int | None):
    """Apply a node relabelling pi (new id of old node v = pi[v]) and an element shuffle sigma
    (new element q = old element sigma[q]); local node order within an element is kept."""
    out = conn
    if elem_seed is not None:
        sigma = torch.from_numpy(seeded_permutation(conn.shape[0], elem_seed)).to(conn.device)
        out = out[sigma]
    if node_seed is not None:
        pi = torch.from_numpy(seeded_permutation(num_nodes, node_seed)).to(conn.device)
        out = pi.to(torch.int32)[out.long()]
    return out.contiguous()


# --------------------------------------------------------------------------------------------
# small random / adversarial meshes (property tests)
# --------------------------------------------------------------------------------------------
def random_mesh(etype: int, num_elems: int, num_nodes: int, seed: int, device=None):
    """Elements with k distinct nodes drawn uniformly from [0, num_nodes) (num_nodes >= k).
    Produces non-manifold edges, isolated nodes and arbitrary orientations."""
    k = ARITY[etype]
    rng = np.random.default_rng(seed)
    conn = np.empty((num_elems, k), dtype=np.int32)
    for e in range(num_elems):
        conn[e] = rng.choice(num_nodes, size=k, replace=False)
    return torch.from_numpy(conn).to(_dev(device)), num_nodes


def nonmanifold_fan(num_tris: int = 3):
    """``num_tris`` triangles sharing edge (0, 1): (0, 1, 2), (0, 1, 3), ...."""
    conn = np.array([[0, 1, 2 + t] for t in range(num_tris)], dtype=np.int32)
    return torch.from_numpy(conn), 2 + num_tris


# --------------------------------------------------------------------------------------------
# polygon / mixed-arity surface meshes: (off int64 [M+1], idx int32 [off[M]], num_nodes); element
# e is the ring idx[off[e]:off[e+1]] (SPEC.md Mesh.element_kind Polygon)
# --------------------------------------------------------------------------------------------
def poly_from_conn(conn: torch.Tensor):
    """A fixed-arity connectivity [M, k] as a polygon mesh (same rings)."""
    M, k = conn.shape
    off = torch.arange(M + 1, device=conn.device, dtype=torch.int64) * k
    return off, conn.reshape(-1).to(torch.int32).contiguous()


def poly_mixed_grid(rows: int, cols: int, seed: int = 1604, device=None):
    """Mixed triangle/quad grid, tri_grid's node numbering.  Cell c = i + cols j becomes, by
    splitmix64(seed)[c] % 3: 0 -> one quad (v00, v10, v11, v01); 1 -> triangles (v00, v10, v11),
    (v00, v11, v01); 2 -> triangles (v00, v10, v01), (v10, v11, v01).  Elements in cell order."""
    d = _dev(device)
    w = cols + 1
    i = torch.arange(cols, device=d, dtype=torch.int64)
    j = torch.arange(rows, device=d, dtype=torch.int64)
    jj, ii = torch.meshgrid(j, i, indexing="ij")
    v00 = (ii + w * jj).reshape(-1)
    v10, v01 = v00 + 1, v00 + w
    v11 = v01 + 1
    ch = torch.from_numpy((splitmix64(seed, rows * cols) % np.uint64(3)).astype(np.int64)).to(d)
    neg = torch.full_like(v00, -1)
    quad = torch.stack([v00, v10, v11, v01, neg, neg], -1)
    t1 = torch.stack([v00, v10, v11, v00, v11, v01], -1)
    t2 = torch.stack([v00, v10, v01, v10, v11, v01], -1)
    slots = torch.where((ch == 0)[:, None], quad, torch.where((ch == 1)[:, None], t1, t2))
    idx = slots.reshape(-1)
    idx = idx[idx >= 0].to(torch.int32).contiguous()
    ar = torch.where((ch == 0)[:, None], torch.tensor([4, 0], device=d), torch.tensor([3, 3], device=d)).reshape(-1)
    ar = ar[ar > 0]
    off = torch.zeros(ar.numel() + 1, dtype=torch.int64, device=d)
    off[1:] = torch.cumsum(ar, 0)
    return off, idx, (rows + 1) * (cols + 1)


def honeycomb(rows: int, cols: int, device=None):
    """Hexagon tiling as a brick wall: hexagon (i, j) (i < cols, j < rows), x = 2i + (j mod 2),
    ring (x, j), (x+1, j), (x+2, j), (x+2, j+1), (x+1, j+1), (x, j+1); node (x, y) -> x + W y,
    W = 2 cols + 2 (a few corner nodes stay isolated).  Interior nodes have 3 neighbours."""
    d = _dev(device)
    W = 2 * cols + 2
    i = torch.arange(cols, device=d, dtype=torch.int64)
    j = torch.arange(rows, device=d, dtype=torch.int64)
    jj, ii = torch.meshgrid(j, i, indexing="ij")
    x = (2 * ii + (jj % 2)).reshape(-1)
    y = jj.reshape(-1)
    ring = torch.stack([x + W * y, x + 1 + W * y, x + 2 + W * y, x + 2 + W * (y + 1), x + 1 + W * (y + 1),
                        x + W * (y + 1)], -1)
    off = torch.arange(rows * cols + 1, device=d, dtype=torch.int64) * 6
    return off, ring.reshape(-1).to(torch.int32).contiguous(), W * (rows + 1)


def random_poly(num_elems: int, num_nodes: int, kmin: int, kmax: int, seed: int, device=None):
    """Polygons of arity uniform in [kmin, kmax] with distinct nodes drawn uniformly from
    [0, num_nodes): non-manifold, isolated nodes, arbitrary orientation."""
    rng = np.random.default_rng(seed)
    ks = rng.integers(kmin, kmax + 1, size=num_elems)
    off = np.zeros(num_elems + 1, dtype=np.int64)
    off[1:] = np.cumsum(ks)
    idx = np.concatenate([rng.choice(num_nodes, size=int(k), replace=False) for k in ks]) if num_elems else \
        np.zeros(0, dtype=np.int64)
    d = _dev(device)
    return torch.from_numpy(off).to(d), torch.from_numpy(idx.astype(np.int32)).to(d), num_nodes


def poly_relabel(off: torch.Tensor, idx: torch.Tensor, num_nodes: int, node_seed: int | None,
                 elem_seed: int | None):
    """relabel() for polygon meshes: node ids through pi, elements reordered by sigma."""
    M = off.numel() - 1
    if elem_seed is not None and M > 0:
        sigma = torch.from_numpy(seeded_permutation(M, elem_seed)).to(off.device)
        ar = (off[1:] - off[:-1])[sigma]
        noff = torch.zeros_like(off)
        noff[1:] = torch.cumsum(ar, 0)
        start = off[:-1][sigma]
        pos = torch.arange(int(noff[-1]), device=off.device) - torch.repeat_interleave(noff[:-1], ar)
        idx = idx[torch.repeat_interleave(start, ar) + pos]
        off = noff
    if node_seed is not None:
        pi = torch.from_numpy(seeded_permutation(num_nodes, node_seed)).to(idx.device)
        idx = pi.to(torch.int32)[idx.long()]
    return off.contiguous(), idx.to(torch.int32).contiguous()


# --------------------------------------------------------------------------------------------
# the five BASELINE.json configs
# --------------------------------------------------------------------------------------------
CONFIGS = {
    1: dict(name="tri_grid_32x32", etype=TRI3,
            desc="2D structured triangle mesh 32x32 cells (2,048 triangles, 1,089 nodes)"),
    2: dict(name="uv_sphere_1000x501", etype=TRI3,
            desc="closed triangulated UV sphere, 1000 lon x 501 rings + 2 poles (1,002,000 tri)"),
    3: dict(name="kuhn_tet_128", etype=TET4,
            desc="Kuhn-subdivided cube tet mesh 128^3 cells (12,582,912 tets)"),
    4: dict(name="hex_256_permuted", etype=HEX8,
            desc="hex mesh 256^3 cells, node labels permuted (seed 1604), elements shuffled (seed 4689)"),
    5: dict(name="kuhn_tet_320", etype=TET4,
            desc="Kuhn tet mesh 320^3 cells (196,608,000 tets)"),
}

# polygon workload (not a BASELINE.json config): mixed tri/quad grid
POLY_CONFIGS = {
    6: dict(name="poly_mixed_8192", desc="mixed triangle/quad polygon grid 8192x8192 cells (seed 1604)"),
}


def make_poly_config(cfg: int, device=None):
    """(off, idx, num_nodes) of a polygon workload."""
    if cfg == 6:
        return poly_mixed_grid(8192, 8192, 1604, device)
    raise ValueError(f"unknown polygon config {cfg}")


def make_config(cfg: int, device=None):
    """Return (etype, conn int32 [M, k], num_nodes) for BASELINE.json config ``cfg`` (1-based)."""
    if cfg == 1:
        conn, n = tri_grid(32, 32, device)
    elif cfg == 2:
        conn, n = uv_sphere(1000, 501, device)
    elif cfg == 3:
        conn, n = kuhn_tets(128, device)
    elif cfg == 4:
        conn, n = hex_grid(256, device)
        conn = relabel(conn, n, 1604, 4689)
    elif cfg == 5:
        conn, n = kuhn_tets(320, device)
    else:
        raise ValueError(f"unknown config {cfg}")
    return CONFIGS[cfg]["etype"], conn, n
