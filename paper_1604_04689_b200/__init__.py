"""paper_1604_04689_b200 — B200-native one-ring nodal neighbours (Mei et al., arXiv 1604.04689).

Thin ctypes binding over ``libmeshnbr.so`` (C ABI: include/meshnbr.h).  Argument marshalling only:
every step of the path runs in the library's sm_100a kernels; torch supplies device memory (its
caching allocator is handed to the library as an ``mn_allocator``), streams and process groups.
There is no CPU fallback: if the library is missing or no CUDA device is present, calls raise.

    import paper_1604_04689_b200 as mn
    offsets, indices = mn.find_node_neighbors(conn_cuda_int32, "tet4", num_nodes)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

__all__ = [
    "TRI3", "QUAD4", "TET4", "HEX8", "MeshError", "lib_path", "load",
    "find_node_neighbors", "find_node_neighbors_sortpairs", "find_node_neighbors_shared", "find_elem_neighbors",
    "find_poly_neighbors", "find_neighbors", "find_neighbors_host", "HostPipeline", "load_off", "load_obj",
    "workspace_bytes", "node_key_bits", "node_key_bytes", "find_neighbors_chunked", "chunk_workspace_bytes",
    "emit_node_pairs", "emit_elem_pairs", "radix_sort_keys", "radix_sort_pairs_u32",
    "unique_node_csr", "elem_offsets", "exclusive_scan",
    "dist_bucket", "dist_finish", "find_neighbors_dist_comm", "find_neighbors_dist_nccl", "find_neighbors_dist_p2p", "symm_create",
    "symm_unmap", "symm_destroy", "dist_plan",
    "alloc_trace", "alloc_trace_take", "trace_peaks",
    "launch_count", "profile_enable", "profile_reset", "profile_collect", "set_elem_path", "get_elem_path", "set_chunk_cap",
]

TRI3, QUAD4, TET4, HEX8 = 0, 1, 2, 3
ARITY = {TRI3: 3, QUAD4: 4, TET4: 4, HEX8: 8}
_NAMES = {"tri3": TRI3, "tri": TRI3, "quad4": QUAD4, "quad": QUAD4, "tet4": TET4, "tet": TET4,
          "hex8": HEX8, "hex": HEX8}

MN_OK, MN_ERR_INVALID_ARG, MN_ERR_INDEX_OUT_OF_RANGE, MN_ERR_DEGENERATE = 0, 1, 2, 3
MN_ERR_CAPACITY, MN_ERR_OOM, MN_ERR_CUDA, MN_ERR_ARITY = 4, 5, 6, 7
MN_ERR_SYNTAX, MN_ERR_COUNT_MISMATCH, MN_ERR_ZERO_INDEX, MN_ERR_COMM = 8, 9, 10, 11

_PKG = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    return os.path.join(_PKG, "libmeshnbr.so")


class MeshError(RuntimeError):
    """Raised for a non-OK mn_status; (code, elem, pos) as in include/meshnbr.h."""

    def __init__(self, code: int, msg: str, elem: int = -1, pos: int = -1):
        super().__init__(f"{msg} (status {code}, elem {elem}, pos {pos})")
        self.code, self.elem, self.pos = code, elem, pos


# ------------------------------------------------------------------------------------------------
# ctypes declarations (mirror include/meshnbr.h)
# ------------------------------------------------------------------------------------------------
_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_RELEASE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class _Allocator(ctypes.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("release", _RELEASE_FN), ("ctx", ctypes.c_void_p)]


class _Csr(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("offsets", ctypes.c_void_p), ("indices", ctypes.c_void_p), ("owner", _Allocator)]


class _HostMesh(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int64), ("num_elems", ctypes.c_int64), ("conn_len", ctypes.c_int64),
                ("off", ctypes.POINTER(ctypes.c_int64)), ("idx", ctypes.POINTER(ctypes.c_int32)),
                ("uniform_arity", ctypes.c_int32)]


class _ErrDetail(ctypes.Structure):
    _fields_ = [("elem", ctypes.c_int64), ("pos", ctypes.c_int32)]


_VP, _I64, _I32, _INT = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
_P = ctypes.POINTER


class A2AOp(ctypes.Structure):
    """mn_a2a_op: one all-to-all(v) of a group (element counts / displacements per rank)."""
    _fields_ = [("send", _VP), ("send_counts", _P(_I64)), ("send_displs", _P(_I64)), ("recv", _VP),
                ("recv_counts", _P(_I64)), ("recv_displs", _P(_I64)), ("elem_bytes", ctypes.c_size_t)]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, _VP, _VP, _VP, ctypes.c_size_t, _VP)
ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, _VP, _P(A2AOp), ctypes.c_int, _VP)


class Comm(ctypes.Structure):
    """mn_comm: the exchange operations of the multi-GPU path (include/meshnbr.h)."""
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("ctx", _VP), ("allgather", ALLGATHER_FN),
                ("alltoallv", ALLTOALLV_FN)]


class DistInfo(ctypes.Structure):
    _fields_ = [("lo", _I64), ("hi", _I64), ("node_base", _I64), ("elem_base", _I64), ("node_nnz_total", _I64),
                ("elem_nnz_total", _I64), ("sent_bytes", _I64), ("recv_bytes", _I64), ("own_incidences", _I64)]


_lib = None


def _declare(lib):
    S = ctypes.c_int
    sig = {
        "mn_find_node_neighbors": (S, [_INT, _VP, _I64, _I64, _P(_Allocator), _VP, _P(_Csr), _P(_ErrDetail)]),
        "mn_find_elem_neighbors": (S, [_INT, _VP, _I64, _I64, _P(_Allocator), _VP, _P(_Csr), _P(_ErrDetail)]),
        "mn_find_node_neighbors_sortpairs": (S, [_INT, _VP, _I64, _I64, _P(_Allocator), _VP, _P(_Csr),
                                                 _P(_ErrDetail)]),
        "mn_find_node_neighbors_shared": (S, [_INT, _VP, _I64, _I64, _P(_Allocator), _VP, _P(_Csr),
                                              _P(_ErrDetail)]),
        "mn_parse_off": (S, [ctypes.c_char_p, ctypes.c_size_t, _P(_HostMesh), _P(_ErrDetail)]),
        "mn_parse_obj": (S, [ctypes.c_char_p, ctypes.c_size_t, _P(_HostMesh), _P(_ErrDetail)]),
        "mn_host_mesh_free": (None, [_P(_HostMesh)]),
        "mn_find_poly_neighbors": (S, [_VP, _VP, _I64, _I64, _I64, _P(_Allocator), _VP, _P(_Csr), _P(_Csr),
                                       _P(_Csr), _P(_ErrDetail)]),
        "mn_find_neighbors_both": (S, [_INT, _VP, _I64, _I64, _P(_Allocator), _VP, _P(_Csr), _P(_Csr),
                                       _P(_ErrDetail)]),
        "mn_host_pipeline_create": (S, [_P(_Allocator), _P(_Allocator), _P(_VP)]),
        "mn_host_pipeline_submit": (S, [_VP, _INT, _VP, _I64, _I64, _P(_Csr), _P(_Csr), _P(_I64), _P(_ErrDetail)]),
        "mn_host_pipeline_wait": (S, [_VP, _I64]),
        "mn_host_pipeline_destroy": (None, [_VP]),
        "mn_find_neighbors_both_host": (S, [_INT, _VP, _I64, _I64, _P(_Allocator), _P(_Allocator), _VP,
                                            _P(_Csr), _P(_Csr), _P(_ErrDetail)]),
        "mn_find_neighbors_both_chunked": (S, [_INT, _VP, _I64, _I64, ctypes.c_size_t, _P(_Allocator), _VP,
                                               _P(_Csr), _P(_Csr), _P(_I64), _P(_ErrDetail)]),
        "mn_chunk_workspace_bytes": (ctypes.c_size_t, [_INT, _I64, _I64, _I64]),
        "mn_csr_release": (None, [_P(_Csr), _VP]),
        "mn_status_string": (ctypes.c_char_p, [_INT]),
        "mn_abi_version": (_INT, []),
        "mn_workspace_bytes": (S, [_INT, _I64, _I64, _INT, _P(ctypes.c_size_t)]),
        "mn_node_key_bits": (_INT, [_I64]),
        "mn_node_key_bytes": (_INT, [_I64]),
        "mn_emit_node_pairs": (S, [_INT, _VP, _I64, _I64, _VP, _VP, _P(_ErrDetail)]),
        "mn_emit_elem_pairs": (S, [_INT, _VP, _I64, _I64, _VP, _VP, _VP, _P(_ErrDetail)]),
        "mn_radix_sort_keys": (S, [_VP, _INT, _I64, _INT, _P(_Allocator), _VP]),
        "mn_radix_sort_pairs_u32": (S, [_VP, _VP, _I64, _INT, _P(_Allocator), _VP]),
        "mn_unique_node_csr": (S, [_VP, _INT, _I64, _I64, _VP, _VP, _P(_I64), _P(_Allocator), _VP]),
        "mn_elem_offsets": (S, [_VP, _I64, _I64, _VP, _VP]),
        "mn_exclusive_scan_i32": (S, [_VP, _I64, _VP, _P(_Allocator), _VP]),
        "mn_dist_bucket": (S, [_INT, _VP, _I64, _I64, _I64, _INT, _INT, _VP, _P(_I64), _P(_VP), _P(_VP),
                               _P(_I64), _P(_Allocator), _VP, _P(_ErrDetail)]),
        "mn_dist_finish": (S, [_INT, _VP, _I64, _VP, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _I64,
                               _P(_Allocator), _VP, _P(_Csr), _P(_Csr)]),
        "mn_find_neighbors_dist": (S, [_INT, _VP, _I64, _I64, _I64, _P(Comm), _P(_Allocator), _VP, _P(_Csr),
                                       _P(_Csr), _P(DistInfo), _P(_ErrDetail)]),
        "mn_find_node_neighbors_dist": (S, [_INT, _VP, _I64, _I64, _I64, _VP, _P(_Allocator), _VP, _P(_Csr),
                                            _P(_I64), _P(_I64), _P(_I64), _P(_ErrDetail)]),
        "mn_find_elem_neighbors_dist": (S, [_INT, _VP, _I64, _I64, _I64, _VP, _P(_Allocator), _VP, _P(_Csr),
                                            _P(_I64), _P(_I64), _P(_I64), _P(_ErrDetail)]),
        "mn_symm_create": (S, [_P(Comm), ctypes.c_size_t, _P(_VP)]),
        "mn_symm_destroy": (S, [_VP]),
        "mn_symm_unmap": (S, [_VP]),
        "mn_symm_capacity": (ctypes.c_size_t, [_VP]),
        "mn_find_neighbors_dist_p2p": (S, [_INT, _VP, _I64, _I64, _I64, _VP, _P(_Allocator), _VP, _P(_Csr),
                                           _P(_Csr), _P(DistInfo), _P(_ErrDetail)]),
        "mn_nccl_available": (_INT, []),
        "mn_nccl_get_unique_id": (S, [_VP]),
        "mn_nccl_comm_init": (S, [_VP, _INT, _INT, _P(_VP)]),
        "mn_nccl_comm_destroy": (S, [_VP]),
        "mn_comm_from_nccl": (S, [_VP, _P(Comm)]),
        "mn_dist_plan": (S, [_INT, _INT, _P(_I64), _P(_I64), _P(_I64), _P(_ErrDetail)]),
        "mn_memcpy_sync": (S, [_VP, _VP, ctypes.c_size_t, _VP]),
        "mn_launch_count": (_I64, []),
        "mn_set_elem_path": (S, [_INT]),
        "mn_get_elem_path": (_INT, []),
        "mn_set_chunk_cap": (S, [_INT]),
        "mn_set_small_path": (S, [_I64]),
        "mn_time_both": (S, [_INT, _VP, _I64, _I64, _INT, _VP, _P(ctypes.c_double), _P(ctypes.c_double)]),
        "mn_profile_enable": (None, [_INT]),
        "mn_profile_reset": (None, []),
        "mn_profile_collect": (_INT, []),
        "mn_profile_entry": (S, [_INT, _P(ctypes.c_char_p), _P(_I64), _P(ctypes.c_double),
                                 _P(ctypes.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """Load libmeshnbr.so (built by __graft_entry__.build() / python -m paper_1604_04689_b200.build).
    Raises if it is missing: there is no fallback path."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_1604_04689_b200.build` "
                              "(nvcc, sm_100a). There is no CPU fallback.")
        lib = ctypes.CDLL(path)
        _declare(lib)
        _lib = lib
    return _lib


# ------------------------------------------------------------------------------------------------
# torch caching allocator -> mn_allocator
# ------------------------------------------------------------------------------------------------
_TRACE = None   # allocation log of the library's device allocations (alloc_trace)


def alloc_trace(enable: bool = True):
    """Start (or stop) logging every device allocation / release the library makes through the
    torch allocator: [("a", ptr, bytes) | ("r", ptr)] in call order (memory-bound checks)."""
    global _TRACE
    _TRACE = [] if enable else None


def alloc_trace_take():
    """The log since alloc_trace(True), and logging stopped."""
    global _TRACE
    t, _TRACE = _TRACE or [], None
    return t


def trace_peaks(trace):
    """From an allocation log: (peak workspace bytes = the most bytes simultaneously live among
    allocations released before the end, peak of the same excluding the allocations still live
    when the last surviving allocation (the last output) was made, output bytes)."""
    size, born, died = {}, {}, {}
    for i, ev in enumerate(trace):
        if ev[0] == "a":
            size[(ev[1], i)] = ev[2]
            born[ev[1]] = (ev[1], i)
        else:
            k = born.pop(ev[1], None)
            if k is not None:
                died[k] = i
    outputs = [k for k in size if k not in died]
    last_out = max((k[1] for k in outputs), default=-1)
    late = {k for k in size if k in died and k[1] < last_out < died[k]}   # e.g. node-index slices
    live = peak = live2 = peak2 = 0
    order = sorted([(k[1], +1, k) for k in size if k in died] + [(died[k], -1, k) for k in died])
    for _, sign, k in order:
        live += sign * size[k]
        peak = max(peak, live)
        if k not in late:
            live2 += sign * size[k]
            peak2 = max(peak2, live2)
    return peak, peak2, sum(size[k] for k in outputs)


class _TorchAllocator:
    """Hands out torch uint8 CUDA tensors; keeps them alive until released or adopted."""

    def __init__(self, device, stream=None):
        self.device = device
        # Blocks come from the caching allocator's pool of the stream the library runs on, so a
        # workspace the library releases while its kernels still read it is only reused by later
        # work on that same stream (stream order), never by the caller's current stream.
        self.stream = stream
        self.live = {}
        self._a = _ALLOC_FN(self._alloc)
        self._r = _RELEASE_FN(self._release)
        self.struct = _Allocator(self._a, self._r, None)

    def _alloc(self, ctx, nbytes, stream):
        try:
            if stream:   # the stream the library allocates on (header: "allocates ... on `stream`")
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device=self.device)):
                    t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
            elif self.stream is not None:
                with torch.cuda.stream(self.stream):
                    t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
            else:
                t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        except RuntimeError:
            return None
        p = t.data_ptr()
        self.live[p] = t
        if _TRACE is not None:
            _TRACE.append(("a", p, int(nbytes)))
        return p

    def _release(self, ctx, ptr, stream):
        if ptr:
            self.live.pop(int(ptr), None)
            if _TRACE is not None:
                _TRACE.append(("r", int(ptr)))

    def adopt(self, ptr, count, dtype):
        """Take ownership of a library output as a typed tensor view."""
        if not ptr or count == 0:
            return torch.empty(0, dtype=dtype, device=self.device)
        t = self.live.pop(int(ptr))
        return t[: count * torch.empty(0, dtype=dtype).element_size()].view(dtype)


class _PinnedAllocator:
    """Host allocator for mn_find_neighbors_both_host: pinned torch CPU tensors."""

    def __init__(self):
        self.live = {}
        self._a = _ALLOC_FN(self._alloc)
        self._r = _RELEASE_FN(self._release)
        self.struct = _Allocator(self._a, self._r, None)

    def _alloc(self, ctx, nbytes, stream):
        t = torch.empty(int(nbytes), dtype=torch.uint8, pin_memory=True)
        self.live[t.data_ptr()] = t
        return t.data_ptr()

    def _release(self, ctx, ptr, stream):
        if ptr:
            self.live.pop(int(ptr), None)

    def adopt(self, ptr, count, dtype):
        if not ptr or count == 0:
            return torch.empty(0, dtype=dtype)
        t = self.live.pop(int(ptr))
        return t[: count * torch.empty(0, dtype=dtype).element_size()].view(dtype)


def _etype(t) -> int:
    if isinstance(t, str):
        return _NAMES[t.lower()]
    t = int(t)
    if t not in ARITY:
        raise ValueError(f"unknown element type {t}")
    return t


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check(rc, err=None):
    if rc != MN_OK:
        msg = load().mn_status_string(rc).decode()
        raise MeshError(rc, msg, err.elem if err is not None else -1, err.pos if err is not None else -1)


def _conn_arg(conn, etype):
    if not isinstance(conn, torch.Tensor) or not conn.is_cuda:
        raise TypeError("conn must be a CUDA tensor (there is no CPU path)")
    if conn.dtype != torch.int32:
        raise TypeError("conn must be int32")
    k = ARITY[etype]
    if conn.numel() % k:
        raise ValueError(f"conn has {conn.numel()} entries, not a multiple of arity {k}")
    return conn.contiguous(), conn.numel() // k


def _take(al, csr):
    n = int(csr.num_nodes)
    off = al.adopt(csr.offsets, n + 1, torch.int64)
    idx = al.adopt(csr.indices, int(csr.nnz), torch.int32)
    return off, idx


# ------------------------------------------------------------------------------------------------
# whole path
# ------------------------------------------------------------------------------------------------
def find_node_neighbors(conn: torch.Tensor, etype, num_nodes: int, stream=None):
    """One-ring neighbouring nodes of every vertex: (offsets int64[N+1], indices int32[nnz])."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    lib = load()
    al = _TorchAllocator(c.device, stream)
    out, err = _Csr(), _ErrDetail()
    with torch.cuda.device(c.device):
        rc = lib.mn_find_node_neighbors(et, c.data_ptr(), M, int(num_nodes), ctypes.byref(al.struct),
                                        _stream_ptr(stream), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return _take(al, out)


def find_node_neighbors_sortpairs(conn: torch.Tensor, etype, num_nodes: int, stream=None):
    """Node CSR by the paper's pipeline verbatim (all node pairs -> global LSD sort -> unique)."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    lib = load()
    al = _TorchAllocator(c.device, stream)
    out, err = _Csr(), _ErrDetail()
    with torch.cuda.device(c.device):
        rc = lib.mn_find_node_neighbors_sortpairs(et, c.data_ptr(), M, int(num_nodes), ctypes.byref(al.struct),
                                                  _stream_ptr(stream), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return _take(al, out)


def find_node_neighbors_shared(conn: torch.Tensor, etype, num_nodes: int, stream=None):
    """Element-sharing node adjacency (u, v neighbours iff some element contains both)."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    lib = load()
    al = _TorchAllocator(c.device, stream)
    out, err = _Csr(), _ErrDetail()
    with torch.cuda.device(c.device):
        rc = lib.mn_find_node_neighbors_shared(et, c.data_ptr(), M, int(num_nodes), ctypes.byref(al.struct),
                                               _stream_ptr(stream), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return _take(al, out)


def find_elem_neighbors(conn: torch.Tensor, etype, num_nodes: int, stream=None):
    """One-ring neighbouring elements of every vertex: (offsets int64[N+1], indices int32[nnz])."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    lib = load()
    al = _TorchAllocator(c.device, stream)
    out, err = _Csr(), _ErrDetail()
    with torch.cuda.device(c.device):
        rc = lib.mn_find_elem_neighbors(et, c.data_ptr(), M, int(num_nodes), ctypes.byref(al.struct),
                                        _stream_ptr(stream), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return _take(al, out)


def find_neighbors(conn: torch.Tensor, etype, num_nodes: int, stream=None):
    """Both CSRs from one call: ((node_offsets, node_indices), (elem_offsets, elem_indices))."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    lib = load()
    al = _TorchAllocator(c.device, stream)
    no, eo, err = _Csr(), _Csr(), _ErrDetail()
    with torch.cuda.device(c.device):
        rc = lib.mn_find_neighbors_both(et, c.data_ptr(), M, int(num_nodes), ctypes.byref(al.struct),
                                        _stream_ptr(stream), ctypes.byref(no), ctypes.byref(eo),
                                        ctypes.byref(err))
    _check(rc, err)
    return _take(al, no), _take(al, eo)


def find_poly_neighbors(off: torch.Tensor, idx: torch.Tensor, num_nodes: int, node: bool = True,
                        elem: bool = True, shared: bool = False, stream=None):
    """Polygon / mixed-arity mesh (element e = ring idx[off[e]:off[e+1]], arity >= 3): any of the
    ring-edge node CSR, the element CSR and the element-sharing node CSR, as (offsets, indices)
    pairs in that order (None where not requested)."""
    for t, dt, nm in ((off, torch.int64, "off"), (idx, torch.int32, "idx")):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{nm} must be a CUDA tensor (there is no CPU path)")
        if t.dtype != dt:
            raise TypeError(f"{nm} must be {dt}")
    if off.numel() < 1:
        raise ValueError("off needs num_elems + 1 entries")
    off, idx = off.contiguous(), idx.contiguous()
    lib = load()
    al = _TorchAllocator(off.device, stream)
    outs = [_Csr() if w else None for w in (node, elem, shared)]
    err = _ErrDetail()
    ref = [ctypes.byref(o) if o is not None else None for o in outs]
    with torch.cuda.device(off.device):
        rc = lib.mn_find_poly_neighbors(off.data_ptr(), idx.data_ptr() if idx.numel() else None, off.numel() - 1,
                                        idx.numel(), int(num_nodes), ctypes.byref(al.struct), _stream_ptr(stream),
                                        *ref, ctypes.byref(err))
    _check(rc, err)
    return tuple(_take(al, o) if o is not None else None for o in outs)


def _parse(fn, data):
    # a path: os.PathLike, or a str holding no line break; any other str is the file's text
    if isinstance(data, os.PathLike) or (isinstance(data, str) and "\n" not in data and "\r" not in data):
        with open(data, "rb") as f:
            data = f.read()
    if isinstance(data, str):
        data = data.encode()
    m, err = _HostMesh(), _ErrDetail()
    rc = fn(data, len(data), ctypes.byref(m), ctypes.byref(err))
    _check(rc, err)
    try:
        M, L = int(m.num_elems), int(m.conn_len)
        off = torch.from_numpy(np.ctypeslib.as_array(m.off, shape=(M + 1,)).copy())
        idx = torch.from_numpy(np.ctypeslib.as_array(m.idx, shape=(L,)).copy() if L else np.zeros(0, np.int32))
        return off, idx, int(m.num_nodes), int(m.uniform_arity)
    finally:
        load().mn_host_mesh_free(ctypes.byref(m))


def load_off(data):
    """Parse an OFF file (path or bytes/str) with the native parser: (off int64[M+1], idx int32,
    num_nodes, uniform_arity) on the host; uniform_arity is k when every face has k nodes, else 0."""
    return _parse(load().mn_parse_off, data)


def load_obj(data):
    """Parse an OBJ file (path or bytes/str); same result as load_off (1-based, negative and
    "/t/n" face tokens resolved)."""
    return _parse(load().mn_parse_obj, data)


def find_neighbors_chunked(conn: torch.Tensor, etype, num_nodes: int, max_workspace_bytes: int, stream=None):
    """Memory-bounded form of find_neighbors: nodes processed in K ranges whose workspace fits in
    max_workspace_bytes.  Returns ((node_offsets, node_indices), (elem_offsets, elem_indices), K)."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    lib = load()
    al = _TorchAllocator(c.device, stream)
    no, eo, err = _Csr(), _Csr(), _ErrDetail()
    k = ctypes.c_int64(0)
    with torch.cuda.device(c.device):
        rc = lib.mn_find_neighbors_both_chunked(et, c.data_ptr(), M, int(num_nodes), int(max_workspace_bytes),
                                                ctypes.byref(al.struct), _stream_ptr(stream), ctypes.byref(no),
                                                ctypes.byref(eo), ctypes.byref(k), ctypes.byref(err))
    _check(rc, err)
    return _take(al, no), _take(al, eo), int(k.value)


def chunk_workspace_bytes(etype, num_elems: int, num_nodes: int, chunks: int) -> int:
    return int(load().mn_chunk_workspace_bytes(_etype(etype), int(num_elems), int(num_nodes), int(chunks)))


def find_neighbors_host(conn_host: torch.Tensor, etype, num_nodes: int, device=None, stream=None):
    """End-to-end form: host (ideally pinned) int32 connectivity in, both CSRs back in pinned host
    memory.  The H2D copy, the kernels and the D2H copies all run inside the library call."""
    et = _etype(etype)
    if conn_host.is_cuda or conn_host.dtype != torch.int32:
        raise TypeError("conn_host must be a host int32 tensor")
    c = conn_host.contiguous()
    M = c.numel() // ARITY[et]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    lib = load()
    dal, hal = _TorchAllocator(dev, stream), _PinnedAllocator()
    no, eo, err = _Csr(), _Csr(), _ErrDetail()
    with torch.cuda.device(dev):
        rc = lib.mn_find_neighbors_both_host(et, c.data_ptr(), M, int(num_nodes), ctypes.byref(dal.struct),
                                             ctypes.byref(hal.struct), _stream_ptr(stream), ctypes.byref(no),
                                             ctypes.byref(eo), ctypes.byref(err))
    _check(rc, err)
    return _take(hal, no), _take(hal, eo)


class HostPipeline:
    """A stream of meshes with host buffers (include/meshnbr.h mn_host_pipeline_*): submit() uploads
    one mesh's connectivity, computes both CSRs and starts their download; wait(ticket) returns them
    as pinned host tensors once the download is complete.  The upload of the next mesh overlaps the
    download of the previous one (PCIe is full duplex).  conn_host must stay unchanged until its
    ticket is waited."""

    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._dal, self._hal = _TorchAllocator(self.device), _PinnedAllocator()
        self._p = ctypes.c_void_p()
        self._lib = load()
        with torch.cuda.device(self.device):
            _check(self._lib.mn_host_pipeline_create(ctypes.byref(self._dal.struct), ctypes.byref(self._hal.struct),
                                                     ctypes.byref(self._p)))
        self._pending = {}

    def submit(self, conn_host: torch.Tensor, etype, num_nodes: int) -> int:
        et = _etype(etype)
        if conn_host.is_cuda or conn_host.dtype != torch.int32:
            raise TypeError("conn_host must be a host int32 tensor")
        c = conn_host.contiguous()
        M = c.numel() // ARITY[et]
        no, eo, err, tk = _Csr(), _Csr(), _ErrDetail(), ctypes.c_int64()
        with torch.cuda.device(self.device):
            rc = self._lib.mn_host_pipeline_submit(self._p, et, c.data_ptr(), M, int(num_nodes), ctypes.byref(no),
                                                   ctypes.byref(eo), ctypes.byref(tk), ctypes.byref(err))
        _check(rc, err)
        self._pending[tk.value] = (c, _take(self._hal, no), _take(self._hal, eo))
        return tk.value

    def wait(self, ticket: int):
        """((node offsets, node indices), (elem offsets, elem indices)) of `ticket`, pinned host tensors."""
        _, node, elem = self._pending.pop(ticket)
        with torch.cuda.device(self.device):
            _check(self._lib.mn_host_pipeline_wait(self._p, int(ticket)))
        return node, elem

    def close(self):
        if self._p:
            with torch.cuda.device(self.device):
                self._lib.mn_host_pipeline_destroy(self._p)
            self._p = ctypes.c_void_p()
            self._pending.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def workspace_bytes(etype, num_elems: int, num_nodes: int, modes: int = 3) -> int:
    out = ctypes.c_size_t(0)
    _check(load().mn_workspace_bytes(_etype(etype), int(num_elems), int(num_nodes), int(modes),
                                     ctypes.byref(out)))
    return int(out.value)


def node_key_bits(num_nodes: int) -> int:
    return int(load().mn_node_key_bits(int(num_nodes)))


def node_key_bytes(num_nodes: int) -> int:
    return int(load().mn_node_key_bytes(int(num_nodes)))


# ------------------------------------------------------------------------------------------------
# stage primitives (one per §8(a) row)
# ------------------------------------------------------------------------------------------------
def emit_node_pairs(conn: torch.Tensor, etype, num_nodes: int, stream=None) -> torch.Tensor:
    """Row a1: packed node-pair keys in creation order (int64 for 8-byte keys, int32 bit pattern
    of uint32 for 4-byte keys)."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    kb = node_key_bytes(num_nodes)
    E = {TRI3: 3, QUAD4: 4, TET4: 6, HEX8: 12}[et]
    keys = torch.empty(2 * E * M, dtype=torch.int64 if kb == 8 else torch.int32, device=c.device)
    err = _ErrDetail()
    with torch.cuda.device(c.device):
        rc = load().mn_emit_node_pairs(et, c.data_ptr(), M, int(num_nodes), keys.data_ptr(),
                                       _stream_ptr(stream), ctypes.byref(err))
    _check(rc, err)
    return keys


def emit_elem_pairs(conn: torch.Tensor, etype, num_nodes: int, stream=None):
    """Row a2: (node keys, element values) in creation order, both int32 tensors."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    n = ARITY[et] * M
    keys = torch.empty(n, dtype=torch.int32, device=c.device)
    vals = torch.empty(n, dtype=torch.int32, device=c.device)
    err = _ErrDetail()
    with torch.cuda.device(c.device):
        rc = load().mn_emit_elem_pairs(et, c.data_ptr(), M, int(num_nodes), keys.data_ptr(), vals.data_ptr(),
                                       _stream_ptr(stream), ctypes.byref(err))
    _check(rc, err)
    return keys, vals


def radix_sort_keys(keys: torch.Tensor, key_bits: int, stream=None) -> torch.Tensor:
    """Row a3: in-place ascending LSD sort of int64 (u64) or int32 (u32 bit pattern) keys."""
    kb = keys.element_size()
    al = _TorchAllocator(keys.device, stream)
    with torch.cuda.device(keys.device):
        rc = load().mn_radix_sort_keys(keys.data_ptr(), kb, keys.numel(), int(key_bits), ctypes.byref(al.struct),
                                       _stream_ptr(stream))
    _check(rc)
    return keys


def radix_sort_pairs_u32(keys: torch.Tensor, vals: torch.Tensor, key_bits: int, stream=None):
    """Row a3e: in-place stable LSD sort of uint32 (key, value) pairs."""
    al = _TorchAllocator(keys.device, stream)
    with torch.cuda.device(keys.device):
        rc = load().mn_radix_sort_pairs_u32(keys.data_ptr(), vals.data_ptr(), keys.numel(), int(key_bits),
                                            ctypes.byref(al.struct), _stream_ptr(stream))
    _check(rc)
    return keys, vals


def unique_node_csr(sorted_keys: torch.Tensor, num_nodes: int, stream=None):
    """Rows a4+a5 (node mode): (offsets int64[N+1], indices int32[nnz]) from sorted packed keys."""
    n = sorted_keys.numel()
    off = torch.empty(int(num_nodes) + 1, dtype=torch.int64, device=sorted_keys.device)
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=sorted_keys.device)
    nnz = ctypes.c_int64(0)
    al = _TorchAllocator(sorted_keys.device, stream)
    with torch.cuda.device(sorted_keys.device):
        rc = load().mn_unique_node_csr(sorted_keys.data_ptr(), sorted_keys.element_size(), n, int(num_nodes),
                                       off.data_ptr(), idx.data_ptr(), ctypes.byref(nnz), ctypes.byref(al.struct),
                                       _stream_ptr(stream))
    _check(rc)
    return off, idx[: nnz.value]


def elem_offsets(sorted_keys: torch.Tensor, num_nodes: int, stream=None) -> torch.Tensor:
    """Rows a4+a5 (element mode): offsets int64[N+1] from stably sorted node keys."""
    off = torch.empty(int(num_nodes) + 1, dtype=torch.int64, device=sorted_keys.device)
    with torch.cuda.device(sorted_keys.device):
        rc = load().mn_elem_offsets(sorted_keys.data_ptr(), sorted_keys.numel(), int(num_nodes), off.data_ptr(),
                                    _stream_ptr(stream))
    _check(rc)
    return off


def exclusive_scan(counts: torch.Tensor, stream=None) -> torch.Tensor:
    """Row a5: int32 counts -> int64 exclusive scan with the total appended (n+1 entries)."""
    out = torch.empty(counts.numel() + 1, dtype=torch.int64, device=counts.device)
    al = _TorchAllocator(counts.device, stream)
    with torch.cuda.device(counts.device):
        rc = load().mn_exclusive_scan_i32(counts.data_ptr(), counts.numel(), out.data_ptr(), ctypes.byref(al.struct),
                                          _stream_ptr(stream))
    _check(rc)
    return out


# ------------------------------------------------------------------------------------------------
# multi-GPU building blocks (orchestrated by paper_1604_04689_b200.dist)
# ------------------------------------------------------------------------------------------------
def dist_bucket(conn_shard: torch.Tensor, etype, global_elem_base: int, num_nodes: int, world: int,
                self_rank: int, stream=None):
    """Bucket this shard's incidences by owner rank.  Returns (pairs int64[k*M] = node << 32 |
    element, counts[world], row_elems int32[R], rows int32[R, k], row_counts[world]): the remote
    rows, one per (destination != self_rank, element), grouped by destination."""
    et = _etype(etype)
    c, M = _conn_arg(conn_shard, et)
    k = ARITY[et]
    pairs = torch.empty(k * M, dtype=torch.int64, device=c.device)
    hc = (ctypes.c_int64 * world)()
    hrc = (ctypes.c_int64 * world)()
    pe, pr = ctypes.c_void_p(), ctypes.c_void_p()
    al = _TorchAllocator(c.device, stream)
    err = _ErrDetail()
    with torch.cuda.device(c.device):
        rc = load().mn_dist_bucket(et, c.data_ptr(), M, int(global_elem_base), int(num_nodes), int(world),
                                   int(self_rank), pairs.data_ptr(), hc, ctypes.byref(pe), ctypes.byref(pr), hrc,
                                   ctypes.byref(al.struct), _stream_ptr(stream), ctypes.byref(err))
    _check(rc, err)
    R = sum(hrc)
    relems = al.adopt(pe.value, R, torch.int32)
    rows = al.adopt(pr.value, R * k, torch.int32).view(R, k)
    return pairs, list(hc), relems, rows, list(hrc)


def dist_finish(etype, pairs: torch.Tensor, row_elems: torch.Tensor, rows: torch.Tensor, conn_shard: torch.Tensor,
                global_elem_base: int, num_nodes: int, lo: int, hi: int, stream=None):
    """CSR slices (node, element) of the owned node range [lo, hi) from the received incidences,
    the received remote rows and the own shard."""
    et = _etype(etype)
    dev = pairs.device
    al = _TorchAllocator(dev, stream)
    ns, es = _Csr(), _Csr()
    rows = rows.contiguous()
    shard = conn_shard.contiguous()
    ptr = lambda t: t.data_ptr() if t.numel() else None  # noqa: E731
    with torch.cuda.device(dev):
        rc = load().mn_dist_finish(et, ptr(pairs), pairs.numel(), ptr(row_elems), ptr(rows), row_elems.numel(),
                                   ptr(shard), shard.numel() // ARITY[et], int(global_elem_base), int(num_nodes),
                                   int(lo), int(hi), ctypes.byref(al.struct), _stream_ptr(stream),
                                   ctypes.byref(ns), ctypes.byref(es))
    _check(rc)
    return _take(al, ns), _take(al, es)


def find_neighbors_dist_comm(conn_shard: torch.Tensor, etype, global_elem_base: int, num_nodes: int, comm: Comm,
                             stream=None):
    """mn_find_neighbors_dist: this rank's node and element CSR slices over the exchange `comm`
    (an mn_comm; see paper_1604_04689_b200.dist for NCCL / gloo ones).  Returns
    (node (offsets, indices), elem (offsets, indices), DistInfo)."""
    et = _etype(etype)
    c, M = _conn_arg(conn_shard, et)
    al = _TorchAllocator(c.device, stream)
    ns, es, info, err = _Csr(), _Csr(), DistInfo(), _ErrDetail()
    with torch.cuda.device(c.device):
        rc = load().mn_find_neighbors_dist(et, c.data_ptr() if M else None, M, int(global_elem_base), int(num_nodes),
                                           ctypes.byref(comm), ctypes.byref(al.struct), _stream_ptr(stream),
                                           ctypes.byref(ns), ctypes.byref(es), ctypes.byref(info), ctypes.byref(err))
    _check(rc, err)
    return _take(al, ns), _take(al, es), info


def symm_create(comm: Comm, initial_bytes: int = 0):
    """mn_symm_create (collective): the symmetric receive heap of the fused P2P path."""
    h = ctypes.c_void_p()
    _check(load().mn_symm_create(ctypes.byref(comm), int(initial_bytes), ctypes.byref(h)))
    return h


def symm_unmap(h):
    _check(load().mn_symm_unmap(h))


def symm_destroy(h):
    _check(load().mn_symm_destroy(h))


def find_neighbors_dist_p2p(conn_shard: torch.Tensor, etype, global_elem_base: int, num_nodes: int, symm,
                            stream=None):
    """mn_find_neighbors_dist_p2p: the fused bucket-and-send path over the symmetric heap `symm`.
    Returns (node (offsets, indices), elem (offsets, indices), DistInfo)."""
    et = _etype(etype)
    c, M = _conn_arg(conn_shard, et)
    al = _TorchAllocator(c.device, stream)
    ns, es, info, err = _Csr(), _Csr(), DistInfo(), _ErrDetail()
    with torch.cuda.device(c.device):
        rc = load().mn_find_neighbors_dist_p2p(et, c.data_ptr() if M else None, M, int(global_elem_base),
                                               int(num_nodes), symm, ctypes.byref(al.struct), _stream_ptr(stream),
                                               ctypes.byref(ns), ctypes.byref(es), ctypes.byref(info),
                                               ctypes.byref(err))
    _check(rc, err)
    return _take(al, ns), _take(al, es), info


def find_neighbors_dist_nccl(conn_shard: torch.Tensor, etype, global_elem_base: int, num_nodes: int, nccl_comm,
                             which: str = "node", stream=None):
    """SURVEY §8(b)'s single-output forms (mn_find_node_neighbors_dist / mn_find_elem_neighbors_dist)
    over a raw ncclComm_t handle.  Returns ((offsets, indices), lo, hi, global_nnz_base)."""
    et = _etype(etype)
    c, M = _conn_arg(conn_shard, et)
    al = _TorchAllocator(c.device, stream)
    out, err = _Csr(), _ErrDetail()
    lo, hi, gb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    fn = load().mn_find_node_neighbors_dist if which == "node" else load().mn_find_elem_neighbors_dist
    with torch.cuda.device(c.device):
        rc = fn(et, c.data_ptr() if M else None, M, int(global_elem_base), int(num_nodes), nccl_comm,
                ctypes.byref(al.struct), _stream_ptr(stream), ctypes.byref(out), ctypes.byref(lo), ctypes.byref(hi),
                ctypes.byref(gb), ctypes.byref(err))
    _check(rc, err)
    return _take(al, out), int(lo.value), int(hi.value), int(gb.value)


def dist_plan(world: int, rank: int, gathered):
    """mn_dist_plan (host only): (status, recv_counts, recv_row_counts, err elem, err pos) from the
    all-gathered int64 rows [error word, status, counts[world], row_counts[world]] of every rank."""
    g = np.ascontiguousarray(np.asarray(gathered, dtype=np.int64).reshape(world, 2 + 2 * world))
    rc = (ctypes.c_int64 * world)()
    rr = (ctypes.c_int64 * world)()
    err = _ErrDetail()
    st = load().mn_dist_plan(int(world), int(rank), g.ctypes.data_as(_P(_I64)), rc, rr, ctypes.byref(err))
    return int(st), list(rc), list(rr), int(err.elem), int(err.pos)


def memcpy_sync(dst: int, src: int, nbytes: int, stream_ptr=None):
    """Copy between raw device / host pointers (cudaMemcpyDefault) on the raw cudaStream_t
    `stream_ptr`, then sync it (used by host-staged exchange callbacks)."""
    _check(load().mn_memcpy_sync(ctypes.c_void_p(dst), ctypes.c_void_p(src), int(nbytes), ctypes.c_void_p(stream_ptr)))


# ------------------------------------------------------------------------------------------------
# instrumentation
# ------------------------------------------------------------------------------------------------
ELEM_PATHS = {"auto": 0, "radix": 1, "transpose": 2, "msd": 3}


def set_elem_path(mode="auto"):
    """Element-CSR algorithm (process-wide): "auto" | "radix" | "transpose" | "msd" (include/meshnbr.h)."""
    _check(load().mn_set_elem_path(ELEM_PATHS[mode] if isinstance(mode, str) else int(mode)))


def set_chunk_cap(cap: int = 0):
    """Test knob: cap the fixed chunk-bucket capacity of the transpose path (0 = auto; include/meshnbr.h)."""
    _check(load().mn_set_chunk_cap(int(cap)))


def time_both(conn: torch.Tensor, etype, num_nodes: int, reps: int = 200, stream=None):
    """mn_time_both: (median, min) host wall microseconds per C-ABI mn_find_neighbors_both call."""
    et = _etype(etype)
    c, M = _conn_arg(conn, et)
    med, mn_ = ctypes.c_double(), ctypes.c_double()
    with torch.cuda.device(c.device):
        _check(load().mn_time_both(et, c.data_ptr(), M, int(num_nodes), int(reps), _stream_ptr(stream),
                                   ctypes.byref(med), ctypes.byref(mn_)))
    return med.value, mn_.value


def set_small_path(max_incidences: int = 8192):
    """One-CTA latency path for small meshes (0 disables; include/meshnbr.h mn_set_small_path)."""
    _check(load().mn_set_small_path(int(max_incidences)))


def get_elem_path() -> str:
    v = int(load().mn_get_elem_path())
    return {b: a for a, b in ELEM_PATHS.items()}[v]


def launch_count() -> int:
    return int(load().mn_launch_count())


def profile_enable(on: bool = True):
    load().mn_profile_enable(1 if on else 0)


def profile_reset():
    load().mn_profile_reset()


def profile_collect():
    """[{name, launches, ms, alg_bytes}] per kernel name since the last reset."""
    lib = load()
    n = lib.mn_profile_collect()
    out = []
    for i in range(n):
        name = ctypes.c_char_p()
        la, ms, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        lib.mn_profile_entry(i, ctypes.byref(name), ctypes.byref(la), ctypes.byref(ms), ctypes.byref(by))
        out.append(dict(name=name.value.decode(), launches=la.value, ms=ms.value, alg_bytes=by.value))
    return out
