"""Oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously correct CPU implementations of what the CUDA path computes, written from
the paper (arxiv 1604.04689, /root/reference/PAPER.md) and SURVEY.md §8(c):

* ``liboracle.so`` (oracle.cpp): the paper's serial baseline — loop over all elements into a
  per-node std::set (node mode) / std::vector (element mode), flattened to CSR.
* ``stages`` (stages.py): the paper's GPU pipeline written out step by step in numpy, in the
  paper's order (pair creation §2.2.1 step 1, sort step 2, segmented reduction + scan step 3),
  one function per step, for per-step parity of the CUDA kernels.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg may
import this package.  The product (paper_1604_04689_b200) never imports it, and it never imports
the product.  Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

OK, ERR_ARG, ERR_RANGE, ERR_DEGENERATE, ERR_ARITY = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile oracle.cpp with plain g++ (no CUDA)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", _SRC, "-o", _SO])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        p64 = ctypes.POINTER(ctypes.c_int64)
        pp64 = ctypes.POINTER(ctypes.POINTER(ctypes.c_int64))
        pp32 = ctypes.POINTER(ctypes.POINTER(ctypes.c_int32))
        p32 = ctypes.POINTER(ctypes.c_int32)
        lib.oracle_validate.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, p64, p32]
        lib.oracle_validate.restype = ctypes.c_int
        for fn in (lib.oracle_node_csr, lib.oracle_elem_csr, lib.oracle_node_shared_csr):
            fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                           pp64, pp32, p64, p64, p32]
            fn.restype = ctypes.c_int
        lib.oracle_poly_validate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                             p64, p32]
        lib.oracle_poly_validate.restype = ctypes.c_int
        lib.oracle_poly_csr.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, pp64, pp32, p64, p64, p32]
        lib.oracle_poly_csr.restype = ctypes.c_int
        lib.oracle_csr_range.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int64, pp64, pp32, p64, p64, p32]
        lib.oracle_csr_range.restype = ctypes.c_int
        lib.oracle_csr_mt.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int, pp64, pp32, p64, p64, p32, p32]
        lib.oracle_csr_mt.restype = ctypes.c_int
        lib.oracle_poly_csr_range.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, pp64, pp32, p64,
                                              p64, p32]
        lib.oracle_poly_csr_range.restype = ctypes.c_int
        lib.oracle_free.argtypes = [ctypes.c_void_p]
        lib.oracle_free.restype = None
        _lib = lib
    return _lib


class OracleMeshError(Exception):
    def __init__(self, code, elem, pos):
        super().__init__(f"oracle: code={code} elem={elem} pos={pos}")
        self.code, self.elem, self.pos = code, elem, pos


def _as_conn(conn) -> np.ndarray:
    if hasattr(conn, "detach"):
        conn = conn.detach().cpu().numpy()
    conn = np.ascontiguousarray(conn, dtype=np.int32)
    return conn


def validate(etype: int, conn, num_nodes: int):
    """(code, elem, pos) of the first invalid element, or (OK, -1, -1)."""
    lib = _load()
    c = _as_conn(conn)
    ee, ep = ctypes.c_int64(-1), ctypes.c_int32(-1)
    rc = lib.oracle_validate(etype, c.ctypes.data, c.shape[0] if c.ndim else 0, num_nodes,
                             ctypes.byref(ee), ctypes.byref(ep))
    return rc, ee.value, ep.value


def _csr(fn, etype, conn, num_nodes):
    lib = _load()
    c = _as_conn(conn)
    M = c.shape[0] if c.size else 0
    off = ctypes.POINTER(ctypes.c_int64)()
    idx = ctypes.POINTER(ctypes.c_int32)()
    nnz = ctypes.c_int64(0)
    ee, ep = ctypes.c_int64(-1), ctypes.c_int32(-1)
    rc = fn(etype, c.ctypes.data, M, num_nodes, ctypes.byref(off), ctypes.byref(idx),
            ctypes.byref(nnz), ctypes.byref(ee), ctypes.byref(ep))
    if rc != OK:
        raise OracleMeshError(rc, ee.value, ep.value)
    offsets = np.ctypeslib.as_array(off, shape=(num_nodes + 1,)).copy()
    indices = (np.ctypeslib.as_array(idx, shape=(nnz.value,)).copy() if nnz.value
               else np.zeros(0, np.int32))
    lib.oracle_free(ctypes.cast(off, ctypes.c_void_p))
    lib.oracle_free(ctypes.cast(idx, ctypes.c_void_p))
    return offsets, indices


def node_csr(etype: int, conn, num_nodes: int):
    """One-ring neighbouring nodes of every vertex as CSR (int64 offsets, int32 indices)."""
    return _csr(_load().oracle_node_csr, etype, conn, num_nodes)


def node_shared_csr(etype: int, conn, num_nodes: int):
    """Element-sharing node adjacency: u, v neighbours iff some element contains both."""
    return _csr(_load().oracle_node_shared_csr, etype, conn, num_nodes)


def elem_csr(etype: int, conn, num_nodes: int):
    """One-ring neighbouring elements of every vertex as CSR (int64 offsets, int32 indices)."""
    return _csr(_load().oracle_elem_csr, etype, conn, num_nodes)


# ---- node-range mode: the same loops restricted to vertices [lo, hi) -----------------
NODE, ELEM, SHARED = 0, 1, 2


def _take(off, idx, nnz, rows):
    offsets = np.ctypeslib.as_array(off, shape=(rows + 1,)).copy()
    indices = (np.ctypeslib.as_array(idx, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int32))
    lib = _load()
    lib.oracle_free(ctypes.cast(off, ctypes.c_void_p))
    lib.oracle_free(ctypes.cast(idx, ctypes.c_void_p))
    return offsets, indices


def csr_range(mode: int, etype: int, conn, num_nodes: int, lo: int, hi: int):
    """CSR slice of vertices [lo, hi): offsets relative to the slice (hi - lo + 1 entries), indices.
    mode NODE (edge adjacency), ELEM (incidence) or SHARED (element-sharing adjacency)."""
    lib = _load()
    c = _as_conn(conn)
    M = c.shape[0] if c.size else 0
    off = ctypes.POINTER(ctypes.c_int64)()
    idx = ctypes.POINTER(ctypes.c_int32)()
    nnz = ctypes.c_int64(0)
    ee, ep = ctypes.c_int64(-1), ctypes.c_int32(-1)
    rc = lib.oracle_csr_range(mode, etype, c.ctypes.data, M, num_nodes, lo, hi, ctypes.byref(off),
                              ctypes.byref(idx), ctypes.byref(nnz), ctypes.byref(ee), ctypes.byref(ep))
    if rc != OK:
        raise OracleMeshError(rc, ee.value, ep.value)
    return _take(off, idx, nnz.value, hi - lo)


def csr_mt(mode: int, etype: int, conn, num_nodes: int, threads: int):
    """Whole CSR from ``threads`` threads, thread t owning vertices [t*N/T, (t+1)*N/T) and scanning
    every element.  -> (offsets, indices, threads actually used)."""
    lib = _load()
    c = _as_conn(conn)
    M = c.shape[0] if c.size else 0
    off = ctypes.POINTER(ctypes.c_int64)()
    idx = ctypes.POINTER(ctypes.c_int32)()
    nnz = ctypes.c_int64(0)
    ee, ep = ctypes.c_int64(-1), ctypes.c_int32(-1)
    used = ctypes.c_int32(0)
    rc = lib.oracle_csr_mt(mode, etype, c.ctypes.data, M, num_nodes, int(threads), ctypes.byref(off),
                           ctypes.byref(idx), ctypes.byref(nnz), ctypes.byref(ee), ctypes.byref(ep),
                           ctypes.byref(used))
    if rc != OK:
        raise OracleMeshError(rc, ee.value, ep.value)
    o, i = _take(off, idx, nnz.value, num_nodes)
    return o, i, used.value


def host_threads() -> int:
    """Host cores this process may run on (the T of the all-core oracle)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---- polygon / mixed-arity meshes: (off int64[M+1], idx int32[off[M]]), ring edges ----
def _as_poly(off, idx):
    if hasattr(off, "detach"):
        off = off.detach().cpu().numpy()
    if hasattr(idx, "detach"):
        idx = idx.detach().cpu().numpy()
    return np.ascontiguousarray(off, dtype=np.int64), np.ascontiguousarray(idx, dtype=np.int32)


def poly_validate(off, idx, num_nodes: int):
    """(code, elem, pos) of the first invalid polygon, or (OK, -1, -1); ERR_ARITY has pos -1."""
    lib = _load()
    o, i = _as_poly(off, idx)
    ee, ep = ctypes.c_int64(-1), ctypes.c_int32(-1)
    rc = lib.oracle_poly_validate(o.ctypes.data, i.ctypes.data, o.shape[0] - 1, num_nodes,
                                  ctypes.byref(ee), ctypes.byref(ep))
    return rc, ee.value, ep.value


def _poly(mode, off, idx, num_nodes):
    lib = _load()
    o, i = _as_poly(off, idx)
    po = ctypes.POINTER(ctypes.c_int64)()
    pi = ctypes.POINTER(ctypes.c_int32)()
    nnz = ctypes.c_int64(0)
    ee, ep = ctypes.c_int64(-1), ctypes.c_int32(-1)
    rc = lib.oracle_poly_csr(mode, o.ctypes.data, i.ctypes.data, o.shape[0] - 1, num_nodes, ctypes.byref(po),
                             ctypes.byref(pi), ctypes.byref(nnz), ctypes.byref(ee), ctypes.byref(ep))
    if rc != OK:
        raise OracleMeshError(rc, ee.value, ep.value)
    offsets = np.ctypeslib.as_array(po, shape=(num_nodes + 1,)).copy()
    indices = (np.ctypeslib.as_array(pi, shape=(nnz.value,)).copy() if nnz.value else np.zeros(0, np.int32))
    lib.oracle_free(ctypes.cast(po, ctypes.c_void_p))
    lib.oracle_free(ctypes.cast(pi, ctypes.c_void_p))
    return offsets, indices


def poly_node_csr(off, idx, num_nodes: int):
    """Ring-edge node adjacency of a polygon mesh as CSR."""
    return _poly(0, off, idx, num_nodes)


def poly_elem_csr(off, idx, num_nodes: int):
    """Element incidence of a polygon mesh as CSR."""
    return _poly(1, off, idx, num_nodes)


def poly_shared_csr(off, idx, num_nodes: int):
    """Element-sharing node adjacency of a polygon mesh as CSR."""
    return _poly(2, off, idx, num_nodes)


def poly_csr_range(mode: int, off, idx, num_nodes: int, lo: int, hi: int):
    """Polygon CSR slice of vertices [lo, hi) (mode NODE / ELEM / SHARED), offsets relative."""
    lib = _load()
    o, i = _as_poly(off, idx)
    po = ctypes.POINTER(ctypes.c_int64)()
    pi = ctypes.POINTER(ctypes.c_int32)()
    nnz = ctypes.c_int64(0)
    ee, ep = ctypes.c_int64(-1), ctypes.c_int32(-1)
    rc = lib.oracle_poly_csr_range(mode, o.ctypes.data, i.ctypes.data, o.shape[0] - 1, num_nodes, lo, hi,
                                   ctypes.byref(po), ctypes.byref(pi), ctypes.byref(nnz), ctypes.byref(ee),
                                   ctypes.byref(ep))
    if rc != OK:
        raise OracleMeshError(rc, ee.value, ep.value)
    return _take(po, pi, nnz.value, hi - lo)


from . import stages  # noqa: E402,F401  (numpy step-by-step oracle)
