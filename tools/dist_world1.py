"""The multi-GPU path at world size 1 (NCCL, one B200): per-call time and per-kernel profile of
mn_find_neighbors_dist (a2a) and _p2p on a workload, against the single-GPU call.  With one rank
everything is owned, so this is the per-rank device work of the path (validation + counts, the
bucket-and-send pass, the finish) without the exchange; at G ranks on a coherent mesh each rank
does this on 1/G of the mesh plus its few remote incidences.

    python tools/dist_world1.py [config]"""
import json
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import meshgen
import paper_1604_04689_b200 as mn
from paper_1604_04689_b200.dist import find_neighbors_dist, release_comms

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
et, conn, N = meshgen.make_config(cfg, device="cuda")
M = conn.shape[0]
ref = mn.find_neighbors(conn, et, N)
out = {"config": cfg, "elements": M}
for name, fn in (("single_gpu", lambda: mn.find_neighbors(conn, et, N)),
                 ("dist_a2a", lambda: find_neighbors_dist(conn, et, 0, N)),
                 ("dist_p2p", lambda: find_neighbors_dist(conn, et, 0, N, p2p=True))):
    for _ in range(3):
        r = fn()
    torch.cuda.synchronize()
    if name != "single_gpu":
        assert torch.equal(r.node[1], ref[0][1]) and torch.equal(r.elem[1], ref[1][1]), name
    del r
    mn.profile_reset(); mn.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        r = fn(); del r
    e1.record(); torch.cuda.synchronize()
    mn.profile_enable(False)
    prof = {e["name"]: round(e["ms"] / 10, 3) for e in mn.profile_collect()}
    out[name] = {"ms": e0.elapsed_time(e1) / 10, "kernels_ms": prof}
print(json.dumps(out))
release_comms()
dist.destroy_process_group()
