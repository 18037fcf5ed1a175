"""Per-kernel device times of mn_find_neighbors_both with the torch caching allocator (the Python
binding) against the library's default allocator (cudaMallocAsync, NULL mn_allocator), config 5."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import meshgen
import paper_1604_04689_b200 as mn
from paper_1604_04689_b200 import _Csr, _ErrDetail, _stream_ptr

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
et, conn, N = meshgen.make_config(cfg, device="cuda")
lib = mn.load()
M = conn.shape[0]


def torch_call():
    r = mn.find_neighbors(conn, et, N)
    del r


def null_call():
    no, eo, err = _Csr(), _Csr(), _ErrDetail()
    s = _stream_ptr(None)
    rc = lib.mn_find_neighbors_both(et, conn.data_ptr(), M, N, None, s, ctypes.byref(no), ctypes.byref(eo),
                                    ctypes.byref(err))
    assert rc == 0
    lib.mn_csr_release(ctypes.byref(no), s)
    lib.mn_csr_release(ctypes.byref(eo), s)


print("mn_time_both (median, min us):", mn.time_both(conn, et, N, reps=20))   # also keeps the default pool's blocks
for name, fn in (("torch", torch_call), ("null", null_call), ("torch", torch_call), ("null", null_call)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 10
    mn.profile_reset(); mn.profile_enable(True)
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    mn.profile_enable(False)
    prof = {e["name"]: e["ms"] / 10 for e in mn.profile_collect()}
    print(f"{name:6s} step {step:.3f} ms  kernels {sum(prof.values()):.3f}  " +
          " ".join(f"{k} {v:.3f}" for k, v in sorted(prof.items(), key=lambda x: -x[1])[:5]), flush=True)
