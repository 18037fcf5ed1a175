"""A/B of node-gather variants (mn_set_gather_variant) on configs 5, 3, 4: per-kernel device times
from the library profiler (CUDA events on the launching stream), bit-equality across variants."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import meshgen
import paper_1604_04689_b200 as mn

variants = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2").split(",")]
cfgs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "5,3,4").split(",")]
mn.load()
for cfg in cfgs:
    et, conn, N = meshgen.make_config(cfg, device="cuda")
    ref = None
    for v in variants:
        mn.set_gather_variant(v)
        for _ in range(3):
            r = mn.find_neighbors(conn, et, N)
        torch.cuda.synchronize()
        if ref is None:
            ref = r
        else:
            same = all(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) for a, b in zip(ref, r))
            assert same, f"variant {v} differs on config {cfg}"
        del r
        mn.profile_reset()
        mn.profile_enable(True)
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            r = mn.find_neighbors(conn, et, N)
            del r
        e1.record(s)
        torch.cuda.synchronize()
        mn.profile_enable(False)
        prof = {e["name"]: e["ms"] / 10 for e in mn.profile_collect()}
        print(f"config {cfg} variant {v}: step {e0.elapsed_time(e1) / 10:.3f} ms  " +
              " ".join(f"{k} {prof[k]:.3f}" for k in ("node_gather", "elem_scatter", "elem_segsort", "node_compact")
                       if k in prof), flush=True)
    mn.set_gather_variant(0)
    del ref, conn
    torch.cuda.empty_cache()
