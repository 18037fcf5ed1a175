"""A/B of library knobs on configs (per-kernel device times from the library profiler, bit-equality
of the outputs across settings).  python tools/ab_knobs.py elem_path 1,2 5,3,4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import meshgen
import paper_1604_04689_b200 as mn

knob = sys.argv[1]
values = [int(x) for x in sys.argv[2].split(",")]
cfgs = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "5,3,4").split(",")]
setter = {"elem_path": lambda v: mn.set_elem_path(int(v)), "small_path": mn.set_small_path}[knob]
mn.load()
for cfg in cfgs:
    et, conn, N = meshgen.make_config(cfg, device="cuda")
    ref = None
    for v in values:
        setter(v)
        for _ in range(4):
            r = mn.find_neighbors(conn, et, N)
        torch.cuda.synchronize()
        if ref is None:
            ref = r
        else:
            assert all(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) for a, b in zip(ref, r)), (knob, v, cfg)
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
        print(f"config {cfg} {knob}={v}: step {e0.elapsed_time(e1) / 10:.3f} ms  " +
              " ".join(f"{k} {prof[k]:.3f}" for k in ("node_gather", "elem_scatter", "elem_segsort", "node_compact")
                       if k in prof), flush=True)
    setter(0)
    del ref, conn
    torch.cuda.empty_cache()
