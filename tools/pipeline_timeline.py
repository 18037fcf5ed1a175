"""Host timeline of the pipelined host API on config 5: submit / wait durations per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import meshgen
import paper_1604_04689_b200 as mn

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
et, conn, N = meshgen.make_config(cfg)
h = conn.contiguous().pin_memory()
pl = mn.HostPipeline()
prev = None
t00 = time.perf_counter()
for k in range(8):
    t0 = time.perf_counter()
    tk = pl.submit(h, et, N)
    t1 = time.perf_counter()
    if prev is not None:
        outs = pl.wait(prev)
        del outs
    t2 = time.perf_counter()
    print(f"step {k}: start {1e3 * (t0 - t00):8.1f} submit {1e3 * (t1 - t0):6.1f} ms  wait(prev) {1e3 * (t2 - t1):6.1f} ms")
    prev = tk
outs = pl.wait(prev)
(no, ni), (eo, ei) = mn.find_neighbors_host(h, et, N)
t0 = time.perf_counter()
for _ in range(3):
    r = mn.find_neighbors_host(h, et, N)
    del r
print(f"single call {1e3 * (time.perf_counter() - t0) / 3:.1f} ms")
