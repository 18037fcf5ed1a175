"""Time mn_find_neighbors_both on every BASELINE config (and both element paths), plus the
paper-literal node path; one JSON line per case (developer tool)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
import paper_1604_04689_b200 as mn  # noqa: E402


def timeit(fn, steps=10, warm=3):
    for _ in range(warm):
        r = fn()
        del r
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        r = fn()
        del r
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for cfg in (1, 2, 3, 4, 5):
    et, conn, N = meshgen.make_config(cfg, device="cuda")
    M = conn.shape[0]
    for path in ("auto", "radix", "transpose"):
        mn.set_elem_path(path)
        ms = timeit(lambda: mn.find_neighbors(conn, et, N))
        print(json.dumps({"config": cfg, "elem_path": path, "elements": M, "ms": ms, "Gelem_per_s": M / ms / 1e6}), flush=True)
    mn.set_elem_path("auto")
    if cfg in (1, 2, 3):
        ms = timeit(lambda: mn.find_node_neighbors_sortpairs(conn, et, N), steps=5)
        print(json.dumps({"config": cfg, "path": "node_sortpairs (paper-literal)", "ms": ms, "Gelem_per_s": M / ms / 1e6}), flush=True)
        ms = timeit(lambda: mn.find_node_neighbors(conn, et, N), steps=5)
        print(json.dumps({"config": cfg, "path": "node only (element-CSR expansion)", "ms": ms, "Gelem_per_s": M / ms / 1e6}), flush=True)
    del conn
    torch.cuda.empty_cache()
