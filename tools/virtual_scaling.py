"""Projected multi-GPU scaling from G virtual ranks on ONE GPU (no NVLink here): every rank's device
work (bucket = validate + owner bucketing + remote rows; finish = element + node CSR slice) is run
in turn on the same GPU and timed with CUDA events; the exchange is not timed but its volume per
rank is counted.  The projection per G is max over ranks of (bucket + finish) + the largest per-rank
exchange over NVLink at the measured 770 GB/s peer bandwidth (B200_PROFILING.md).  A projection,
not a measurement of N > 1.

    python tools/virtual_scaling.py [config] [G list]   -> one JSON line per G
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import meshgen
import paper_1604_04689_b200 as mn
from paper_1604_04689_b200.dist import owner_range

NVLINK_GBPS = 770.0


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(cfg, G, reps=3):
    et, conn, N = meshgen.make_config(cfg, device="cuda")
    M = conn.shape[0]
    k = meshgen.ARITY[et]
    best = None
    for _ in range(reps):
        sent, shards, tb = [], [], []
        for r in range(G):
            s0, s1 = r * M // G, (r + 1) * M // G
            shard = conn[s0:s1].contiguous()
            a, b = ev(), ev()
            a.record()
            pairs, cnt, relems, rows, rcnt = mn.dist_bucket(shard, et, s0, N, G, r)
            b.record()
            torch.cuda.synchronize()
            tb.append(a.elapsed_time(b))
            sent.append((list(torch.split(pairs, cnt)), list(torch.split(relems, rcnt)),
                         list(torch.split(rows, rcnt)), cnt, rcnt))
            shards.append((shard, s0))
        tf, xbytes = [], []
        for g in range(G):
            lo, hi = owner_range(N, G, g)
            pin = torch.cat([sent[r][0][g] for r in range(G)])
            ein = torch.cat([sent[r][1][g] for r in range(G)])
            rin = torch.cat([sent[r][2][g] for r in range(G)])
            a, b = ev(), ev()
            a.record()
            out = mn.dist_finish(et, pin, ein, rin, shards[g][0], shards[g][1], N, lo, hi)
            b.record()
            torch.cuda.synchronize()
            tf.append(a.elapsed_time(b))
            del out, pin, ein, rin
            recv = sum(sent[r][3][g] * 8 + sent[r][4][g] * 4 * (k + 1) for r in range(G) if r != g)
            send = sum(sent[g][3][h] * 8 + sent[g][4][h] * 4 * (k + 1) for h in range(G) if h != g)
            xbytes.append((send, recv))
        per_rank = [tb[i] + tf[i] for i in range(G)]
        xmax = max(max(s, r) for s, r in xbytes)
        proj = max(per_rank) + xmax / (NVLINK_GBPS * 1e9) * 1e3
        line = {"config": cfg, "G": G, "elements": M, "bucket_ms": tb, "finish_ms": tf,
                "max_rank_ms": max(per_rank), "exchange_bytes_max": xmax,
                "remote_fraction": sum(s for s, _ in xbytes) / max(1, 8 * k * M + 0.0),
                "projected_ms": proj, "projected_elements_per_s": M / (proj / 1e3)}
        if best is None or line["projected_ms"] < best["projected_ms"]:
            best = line
        del sent, shards
        torch.cuda.empty_cache()
    return best


if __name__ == "__main__":
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    Gs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
    mn.load()
    for G in Gs:
        print(json.dumps(run(cfg, G)), flush=True)
