#!/usr/bin/env python
"""Benchmark: mesh elements/s to CSR node + element one-ring neighbours (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the whole hot path (both modes) over the
workload: at N=1 the whole of config 5 (Kuhn tets 320^3, 196,608,000 tets) on one GPU; at N>1
config 5 sharded by elements over N ranks with the NCCL all-to-all (strong scaling: the same
mesh).  Inputs are resident in HBM before the timed region and larger than L2 (3.15 GB of
connectivity, 18.9 GB of node keys), so no explicit L2 flush is needed.  One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mesh elements/sec to CSR node+elem neighbors; achieved HBM GB/s vs peak, 1/2/4/8 GPU"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--outputs", default="both", choices=["both", "shared"],
                    help="both = node + element CSR (the headline); shared = element-sharing node "
                         "adjacency (SURVEY §8(f) row 3), N=1 only")
    ap.add_argument("--max-workspace-gb", type=float, default=None,
                    help="memory-bounded mode (SURVEY §8(f) row 4): node ranges whose workspace fits this budget")
    ap.add_argument("--elem-path", default="auto", choices=["auto", "radix", "transpose"],
                    help="element-CSR algorithm (auto = locality test; see DESIGN.md §3.5)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "a2a"],
                    help="N>1: p2p = fused bucket-and-send into the owners' symmetric heaps over peer memory "
                         "(mn_find_neighbors_dist_p2p); a2a = bucket, NCCL all-to-all, finish (mn_find_neighbors_dist)")
    ap.add_argument("--cpu-seconds", type=float, default=16.0, help="target oracle sample time")
    ap.add_argument("--no-parity", action="store_true", help="skip the pre-timing parity gate (profiling only)")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
# helpers
# ------------------------------------------------------------------------------------------------
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []          # (host time, csv line)
        self.window = None       # (t0, t1) of the timed region, host clock

    def __enter__(self):
        if os.environ.get("MN_BENCH_NO_CLOCKS"):   # (diagnostics only: a line without clocks is not a result)
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) can stall CUDA calls for tens of ms: wait until it has
            # produced samples before the timed region starts
            t0 = time.time()
            while len(self.lines) < 2 and time.time() - t0 < 10:
                time.sleep(0.02)
            time.sleep(0.1)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ts, ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), float(f[3]), f[4:8], ts))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        if self.window:
            t0, t1 = self.window
            inside = [r for r in rows if t0 <= r[4] <= t1]
            if len(inside) < 3:   # a short timed region: the samples nearest to it
                mid = 0.5 * (t0 + t1)
                inside = sorted(rows, key=lambda r: abs(r[4] - mid))[:3]
            rows = inside
        pmax = max(r[2] for r in rows)
        load = rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(load), "power_w_max": pmax}


def workload(cfg, rank, world, device):
    """(etype, conn shard on device, global element base, total elements, num_nodes, desc)."""
    import meshgen
    if cfg in meshgen.POLY_CONFIGS:   # polygon workload: etype None, conn = (off, idx)
        if world > 1:
            raise SystemExit("polygon configs are single-GPU")
        off, idx, N = meshgen.make_poly_config(cfg, device=device)
        info = dict(meshgen.POLY_CONFIGS[cfg], etype=None)
        return None, (off, idx), 0, off.numel() - 1, N, info
    info = meshgen.CONFIGS[cfg]
    if cfg in (3, 5) and world > 1:
        n = 128 if cfg == 3 else 320
        ncell = n ** 3
        c0, c1 = rank * ncell // world, (rank + 1) * ncell // world
        conn, N = meshgen.kuhn_tets(n, device=device, cell_begin=c0, cell_end=c1)
        return info["etype"], conn, 6 * c0, 6 * ncell, N, info
    et, conn, N = meshgen.make_config(cfg, device=device)
    M = conn.shape[0]
    if world > 1:
        s0, s1 = rank * M // world, (rank + 1) * M // world
        return et, conn[s0:s1].contiguous(), s0, M, N, info
    return et, conn, 0, M, N, info


def oracle_sample(conn_full_dev, et, target_s, k_layers_hint=None, outputs="both", threads=1):
    """Time the oracle (std::set serial baseline; with threads > 1 its T-thread node-range mode,
    SURVEY §8(c)) on a bounded prefix of the workload: the first Ms elements with N trimmed to the
    largest node id + 1.  Returns (elements/s, description, seconds, Ms)."""
    import numpy as np

    import oracle
    if et is not None and threads > 1:
        M = conn_full_dev.shape[0]
        ms = min(M, 500_000)
        modes = [oracle.SHARED] if outputs == "shared" else [oracle.NODE, oracle.ELEM]
        while True:
            sub = conn_full_dev[:ms].cpu().numpy()
            n_s = int(sub.max()) + 1 if sub.size else 0
            t0 = time.perf_counter()
            for m in modes:
                _, _, used = oracle.csr_mt(m, et, sub, n_s, threads)
            dt = time.perf_counter() - t0
            what = "element-sharing node CSR" if outputs == "shared" else "node + element CSR"
            if dt >= 0.6 * target_s or ms >= M:
                return ms / dt, (f"first {ms:,} of {M:,} elements (node ids < {n_s:,}), {what}, "
                                 f"{used} threads (node-range mode), {dt:.1f} s"), dt, ms
            ms = min(M, int(ms * max(1.5, min(8.0, target_s / max(dt, 1e-3)))))
    if et is None:   # polygon workload
        off_d, idx_d = conn_full_dev
        M = off_d.numel() - 1
        ms = min(M, 200_000)
        while True:
            off = off_d[:ms + 1].cpu().numpy()
            idx = idx_d[:int(off[-1])].cpu().numpy()
            n_s = int(idx.max()) + 1 if idx.size else 0
            t0 = time.perf_counter()
            if outputs == "shared":
                oracle.poly_shared_csr(off, idx, n_s)
            else:
                oracle.poly_node_csr(off, idx, n_s)
                oracle.poly_elem_csr(off, idx, n_s)
            dt = time.perf_counter() - t0
            what = "element-sharing node CSR" if outputs == "shared" else "node + element CSR"
            if dt >= 0.6 * target_s or ms >= M:
                return ms / dt, (f"first {ms:,} of {M:,} polygons (node ids < {n_s:,}), {what}, "
                                 f"1 thread, {dt:.1f} s"), dt, ms
            ms = min(M, int(ms * max(1.5, min(8.0, target_s / max(dt, 1e-3)))))
    M = conn_full_dev.shape[0]
    ms = min(M, 200_000)
    while True:
        sub = conn_full_dev[:ms].cpu().numpy()
        n_s = int(sub.max()) + 1 if sub.size else 0
        t0 = time.perf_counter()
        if outputs == "shared":
            oracle.node_shared_csr(et, sub, n_s)
        else:
            oracle.node_csr(et, sub, n_s)
            oracle.elem_csr(et, sub, n_s)
        dt = time.perf_counter() - t0
        what = "element-sharing node CSR" if outputs == "shared" else "node + element CSR"
        if dt >= 0.6 * target_s or ms >= M:
            return ms / dt, (f"first {ms:,} of {M:,} elements (node ids < {n_s:,}), {what}, "
                             f"1 thread, {dt:.1f} s"), dt, ms
        ms = min(M, int(ms * max(1.5, min(8.0, target_s / max(dt, 1e-3)))))


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _slice(csr, lo, a, b):
    """Rows [a, b) of a device CSR whose first row is vertex lo -> host (relative offsets, indices)."""
    off, idx = csr
    o = off[a - lo:b - lo + 1].cpu().numpy()
    i = idx[int(o[0]):int(o[-1])].cpu().numpy() if o.size else idx[:0].cpu().numpy()
    return o - (o[0] if o.size else 0), i


def parity_gate(et, conn_cpu, N, outs, lo=0, hi=None, rows=1 << 15):
    """Bit-exact comparison of the timed call's outputs with the oracle's node-range mode (SURVEY
    §8(c)) on three vertex ranges (first, middle, last of [lo, hi)), before any timing is printed
    (SPEC S:L418, L435).  outs: {oracle mode: device CSR whose first row is vertex lo}.
    Raises SystemExit on a mismatch.  -> description of what was checked."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle
    hi = N if hi is None else hi
    R = min(rows, hi - lo)
    ranges = sorted({(lo, lo + R), ((lo + hi - R) // 2, (lo + hi + R) // 2), (hi - R, hi)})
    jobs = []
    with ThreadPoolExecutor(max_workers=len(ranges) * len(outs)) as ex:   # ctypes releases the GIL
        for mode, csr in outs.items():
            for a, b in ranges:
                if et is None:
                    fut = ex.submit(oracle.poly_csr_range, mode, conn_cpu[0], conn_cpu[1], N, a, b)
                else:
                    fut = ex.submit(oracle.csr_range, mode, et, conn_cpu, N, a, b)
                jobs.append((mode, a, b, csr, fut))
        nv = 0
        for mode, a, b, csr, fut in jobs:
            ro, ri = fut.result()
            go, gi = _slice(csr, lo, a, b)
            if not (np.array_equal(go, ro) and np.array_equal(gi, ri)):
                raise SystemExit(f"parity gate FAILED: mode {mode}, vertices [{a}, {b}) differ from the oracle; "
                                 "no timing reported")
            nv += b - a
    names = {0: "node", 1: "elem", 2: "shared"}
    return {"ok": True, "oracle": "node-range mode (oracle/oracle.cpp oracle_csr_range)",
            "outputs": [names[m] for m in outs], "vertex_ranges": [list(r) for r in ranges],
            "vertices_checked_per_output": sum(b - a for a, b in ranges), "compare": "bit-exact (memcmp)"}


# ------------------------------------------------------------------------------------------------
# reference arm: the oracle, timed as it stands on the host cores
# ------------------------------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch

    import meshgen
    import oracle
    if args.config in meshgen.POLY_CONFIGS:
        return run_reference_poly(args)
    if args.config == 5:   # only the leading cell layers are ever sampled: build just those
        et, conn = meshgen.TET4, meshgen.kuhn_tets(320, cell_begin=0, cell_end=320 * 320 * 128)[0]
        M_total, N_total = 6 * 320 ** 3, 321 ** 3
    else:
        et, conn, N_total = meshgen.make_config(args.config, device="cpu")
        M_total = int(conn.shape[0])
    conn = conn.numpy()
    T = oracle.host_threads()   # the oracle's T-thread node-range mode on all host cores

    def one(sub, n_s):
        oracle.csr_mt(oracle.NODE, et, sub, n_s, T)
        oracle.csr_mt(oracle.ELEM, et, sub, n_s, T)

    # size the per-step sample for ~ (few minutes) / (steps + warmup)
    per_step = max(1.0, min(20.0, 150.0 / (args.steps + args.warmup)))
    ms = min(conn.shape[0], 100_000)
    while True:
        sub = conn[:ms]
        n_s = int(sub.max()) + 1
        t0 = time.perf_counter()
        one(sub, n_s)
        dt = time.perf_counter() - t0
        if dt >= 0.6 * per_step or ms >= conn.shape[0]:
            break
        ms = min(conn.shape[0], int(ms * max(1.5, min(8.0, per_step / max(dt, 1e-3)))))
    sub = conn[:ms]
    n_s = int(sub.max()) + 1
    for _ in range(args.warmup):
        one(sub, n_s)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one(sub, n_s)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = ms / t
    sample = (f"first {ms:,} elements of config {args.config} ({meshgen.CONFIGS[args.config]['name']}), "
              f"node ids < {n_s:,}; std::set oracle, node + element CSR, {T} threads (node-range mode, "
              f"{cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"config {args.config}: {meshgen.CONFIGS[args.config]['desc']}",
                       "elements": M_total, "nodes": N_total, "parallelism": f"host, {T} threads (oracle)",
                       "outputs": "node + element CSR", "sample_elements": ms},
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": T, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def run_reference_poly(args):
    """Reference arm on a polygon workload: the oracle's polygon functions on a prefix sample."""
    import meshgen
    import oracle
    off_t, idx_t, N_total = meshgen.make_poly_config(args.config, device="cpu")
    off_all, idx_all = off_t.numpy(), idx_t.numpy()
    M = off_all.shape[0] - 1
    per_step = max(1.0, min(20.0, 150.0 / (args.steps + args.warmup)))

    def sample(ms):
        off = off_all[:ms + 1]
        idx = idx_all[:int(off[-1])]
        return off, idx, int(idx.max()) + 1

    def one(off, idx, n_s):
        oracle.poly_node_csr(off, idx, n_s)
        oracle.poly_elem_csr(off, idx, n_s)

    ms = min(M, 100_000)
    while True:
        t0 = time.perf_counter()
        one(*sample(ms))
        dt = time.perf_counter() - t0
        if dt >= 0.6 * per_step or ms >= M:
            break
        ms = min(M, int(ms * max(1.5, min(8.0, per_step / max(dt, 1e-3)))))
    off, idx, n_s = sample(ms)
    for _ in range(args.warmup):
        one(off, idx, n_s)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one(off, idx, n_s)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = ms / t
    sample_desc = (f"first {ms:,} polygons of config {args.config} ({meshgen.POLY_CONFIGS[args.config]['name']}), "
                   f"node ids < {n_s:,}; std::set oracle, node + element CSR, 1 thread")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"config {args.config}: {meshgen.POLY_CONFIGS[args.config]['desc']}",
                       "elements": M, "nodes": int(N_total),
                       "parallelism": "host, 1 thread (oracle)", "outputs": "node + element CSR",
                       "sample_elements": ms},
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": 1, "kind": "oracle",
                             "sample": sample_desc},
            "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1604_04689_b200 as mn
    from paper_1604_04689_b200 import build as mnbuild

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    local = local % max(1, torch.cuda.device_count())   # several test ranks may share one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        mnbuild.build()
    if world > 1:
        # MN_DIST_BACKEND=gloo stages the exchange through host memory: it lets several ranks share
        # one GPU to exercise this path in tests; the product exchange is NCCL over NVLink
        backend = os.environ.get("MN_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        dist.barrier()
    mn.load()
    mn.set_elem_path(args.elem_path)

    et, conn, base, M_total, N, info = workload(args.config, rank, world, dev)
    poly = et is None
    torch.cuda.synchronize()

    if poly:
        shared = args.outputs == "shared"

        def step():
            return mn.find_poly_neighbors(conn[0], conn[1], N, node=not shared, elem=not shared, shared=shared)
    elif args.outputs == "shared":
        if world > 1:
            raise SystemExit("--outputs shared is single-GPU")

        def step():
            return mn.find_node_neighbors_shared(conn, et, N)
    elif world > 1:
        from paper_1604_04689_b200.dist import find_neighbors_dist, symm_for
        use_p2p = args.exchange == "p2p"
        if use_p2p:
            try:
                symm_for()          # collective: the symmetric heaps, mapped on every rank
            except mn.MeshError as e:
                print(f"p2p exchange unavailable ({e}); using the NCCL all-to-all", file=sys.stderr)
                use_p2p = False

        def step():
            return find_neighbors_dist(conn, et, base, N, p2p=use_p2p)
    elif args.max_workspace_gb:
        budget = int(args.max_workspace_gb * 2**30)
        chunks_used = []

        def step():
            no, eo, k = mn.find_neighbors_chunked(conn, et, N, budget)
            chunks_used.append(k)
            return no, eo
    else:
        def step():
            return mn.find_neighbors(conn, et, N)

    def barrier():
        if world > 1:
            dist.barrier()

    def maxover(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    mem_bound = None
    if args.max_workspace_gb and not poly and world == 1:   # measured peak of the bounded mode
        torch.cuda.synchronize()
        mn.alloc_trace(True)
        rr = step()
        torch.cuda.synchronize()
        peak, peak_ws, outb = mn.trace_peaks(mn.alloc_trace_take())
        del rr
        mem_bound = {"max_workspace_bytes": int(args.max_workspace_gb * 2**30), "peak_workspace_bytes": peak_ws,
                     "peak_with_node_slices_bytes": peak, "output_bytes": outb,
                     "node_ranges": chunks_used[-1],
                     "source": "library allocation log (paper_1604_04689_b200.alloc_trace)"}

    # ---- parity gate: one more call, its outputs compared with the oracle's
    # node-range mode before anything is timed; also gives the output sizes for B_min ----
    r = step()
    torch.cuda.synchronize()
    parity = None
    nnz = {}
    if poly:
        node_r, elem_r, shared_r = r
        outs = {m: c for m, c in ((0, node_r), (1, elem_r), (2, shared_r)) if c is not None}
    elif args.outputs == "shared":
        outs = {2: r}
    elif world > 1:
        outs = {0: r.node, 1: r.elem}
    else:
        outs = {0: r[0], 1: r[1]}
    for m, c in outs.items():
        nnz[m] = int(c[1].numel())
    exchange = None
    if world > 1:   # slices: total nnz over ranks; exchange volume (SURVEY §8(d) multi-GPU model)
        nnz = {0: r.node_nnz_total, 1: r.elem_nnz_total}
        x = torch.tensor([r.sent_bytes, r.recv_bytes, r.own_incidences], dtype=torch.int64,
                         device=dev if dist.get_backend() == "nccl" else "cpu")
        xs = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(xs, x)
        xs = torch.stack(xs).cpu().tolist()
        exchange = {"mode": "p2p: bucketing kernel stores into the owners' symmetric heaps (NVLink peer memory)"
                            if use_p2p else "a2a: bucket, one grouped NCCL all-to-all, finish",
                    "payload": ("remote incidence 8 B + its element row 4k B" if use_p2p else
                                "remote (node, element) incidence 8 B + remote element id and row 4(k+1) B")
                               + "; own incidences stay in place",
                    "sent_bytes_per_rank": [v[0] for v in xs], "recv_bytes_per_rank": [v[1] for v in xs],
                    "own_incidence_fraction": sum(v[2] for v in xs) / max(1, nnz[1]),
                    "backend": dist.get_backend()}
    if not args.no_parity and rank == 0:
        if world > 1:   # rank 0 checks its own slice against the whole mesh (built on the host)
            import meshgen
            _, conn_full, _ = meshgen.make_config(args.config, device="cpu")
            parity = parity_gate(et, conn_full.numpy(), N, outs, lo=r.lo, hi=r.hi)
            del conn_full
        elif poly:
            parity = parity_gate(None, (conn[0].cpu().numpy(), conn[1].cpu().numpy()), N, outs)
        else:
            parity = parity_gate(et, conn.cpu().numpy(), N, outs)
    if world > 1:
        dist.barrier()
    del r, outs
    torch.cuda.synchronize()

    # warm-up after the parity gate / allocation-log calls, so the caching allocator is back in its
    # steady state when the timed region starts (its first step must not pay a cudaMalloc)
    for _ in range(args.warmup):
        r = step()
        del r
    torch.cuda.synchronize()

    # ---- device-timed region ----
    s = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mn.profile_reset()
    mn.profile_enable(True)
    launches0 = mn.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_host0 = time.time()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        mstat0 = torch.cuda.memory_stats(dev)
        ev0.record(s)
        for i in range(args.steps):
            r = step()
            del r
            evs[i].record(s)
        ev1.record(s)
        torch.cuda.synchronize()
        clk.window = (t_host0, time.time())
    step_seq = [ev0.elapsed_time(evs[0])] + [evs[i - 1].elapsed_time(evs[i]) for i in range(1, args.steps)]
    step_ms = sorted(step_seq)
    if os.environ.get("MN_BENCH_STEPS"):
        ms_now = torch.cuda.memory_stats(dev)
        print("steps", [round(x, 3) for x in step_seq],
              {k: ms_now.get(k, 0) - mstat0.get(k, 0) for k in ("num_device_alloc", "num_device_free", "num_alloc_retries")},
              file=sys.stderr)
    barrier()
    launches = mn.launch_count() - launches0
    mn.profile_enable(False)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = maxover(ms_local)
    prof = mn.profile_collect()
    mn.profile_reset()
    value = M_total / (ms / 1e3)

    # ---- latency of one call (small configs are launch/latency-bound: report microseconds) ----
    latency = None
    if world == 1 and not poly and args.outputs == "both" and not args.max_workspace_gb and M_total <= 20_000_000:
        reps = 300 if M_total <= 100_000 else 50
        c_med, c_min = mn.time_both(conn, et, N, reps=reps)
        walls = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = mn.find_neighbors(conn, et, N)
            torch.cuda.current_stream().synchronize()
            walls.append((time.perf_counter() - t0) * 1e6)
            del r
        walls.sort()
        latency = {"c_abi_median_us": c_med, "c_abi_min_us": c_min, "python_median_us": walls[len(walls) // 2],
                   "reps": reps, "what": "host wall time per call, from entry until both CSRs are complete on the "
                                         "stream (C ABI: mn_time_both, default allocator, stream sync included; "
                                         "python: find_neighbors + sync)"}

    # ---- roofline of the dominant kernel (live CUDA events on the launching stream) ----
    peak, peak_src = peaks()
    prof = sorted(prof, key=lambda e: -e["ms"])
    top = prof[0]
    achieved = (top["alg_bytes"] / top["launches"]) / ((top["ms"] / top["launches"]) / 1e3) / 1e9
    tot_ms = sum(e["ms"] for e in prof)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"config{args.config}/n{world}/{top['name']}")
    step_bytes = sum(e["alg_bytes"] for e in prof) / args.steps
    roofline = {"bound": "hbm", "kernel": top["name"], "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": top["alg_bytes"] / top["launches"],
                "avg_launch_ms": top["ms"] / top["launches"],
                "share_of_kernel_time": top["ms"] / tot_ms if tot_ms else None}
    # secondary: the same kernel against the instruction-issue roofline (warp instructions per launch
    # from a committed ncu capture, profiles/issue.json; 148 SMs x 4 schedulers x sm clock)
    ip = os.path.join(ROOT, "profiles", "issue.json")
    if os.path.exists(ip) and args.outputs == "both" and not args.max_workspace_gb:   # (the captured path only)
        inst = json.load(open(ip)).get(f"config{args.config}/n{world}/{top['name']}")
        if inst:
            clk_mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0)) \
                if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
            ipeak = 148 * 4 * clk_mhz * 1e6
            iach = inst / (roofline["avg_launch_ms"] / 1e3)
            roofline["issue"] = {"warp_instructions_per_launch": inst, "achieved_per_s": iach,
                                 "peak_per_s": ipeak, "frac": iach / ipeak,
                                 "source": "ncu smsp__inst_executed.sum (profiles/issue.json); peak = 148 SMs x 4 "
                                           "issue slots x sm_max clock"}
    kernels = [{"name": e["name"], "launches_per_step": e["launches"] / args.steps,
                "ms_per_step": e["ms"] / args.steps, "share": e["ms"] / tot_ms if tot_ms else None,
                "GBps": (e["alg_bytes"] / (e["ms"] / 1e3) / 1e9) if e["ms"] > 0 else None} for e in prof]
    step_roof = {"step_ms_min_median_max": [step_ms[0], step_ms[len(step_ms) // 2], step_ms[-1]],
                 "alg_bytes_per_step": step_bytes, "achieved_GBps": step_bytes / (ms_local / 1e3) / 1e9,
                 "frac_of_peak": step_bytes / (ms_local / 1e3) / 1e9 / peak,
                 "kernel_ms_per_step": tot_ms / args.steps}
    # compulsory floor: connectivity read once, every output written once
    if poly:
        conn_bytes = conn[0].numel() * 8 + conn[1].numel() * 4
    else:
        conn_bytes = conn.numel() * 4 * (world if world > 1 else 1)   # (shards: approximately the mesh)
    b_min = conn_bytes + sum(4 * v + 8 * (N + 1) for v in nnz.values())
    step_roof.update({"B_min_bytes": b_min, "B_min_GBps": b_min / (ms / 1e3) / 1e9,
                      "frac_vs_B_min": b_min / (ms / 1e3) / 1e9 / peak,
                      "B_min_def": "connectivity once + each output CSR once (int32 indices, int64 offsets)"})

    # ---- end to end through the public host-buffer API ----
    e2e = None
    if not args.no_e2e and args.outputs == "both" and not args.max_workspace_gb:
        host_conn = (conn[0].cpu().pin_memory(), conn[1].cpu().pin_memory()) if poly else conn.cpu().pin_memory()
        h2d = (host_conn[0].numel() * 8 + host_conn[1].numel() * 4) if poly else host_conn.numel() * 4

        if poly:
            def estep():
                o = host_conn[0].to(dev, non_blocking=True)
                i = host_conn[1].to(dev, non_blocking=True)
                (no, ni), (eo, ei), _ = mn.find_poly_neighbors(o, i, N, node=True, elem=True)
                outs = []
                for x in (no, ni, eo, ei):   # pinned (torch's caching host allocator), async D2H
                    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
                    h.copy_(x, non_blocking=True)
                    outs.append(h)
                torch.cuda.current_stream().synchronize()
                return outs
        elif world > 1:
            from paper_1604_04689_b200.dist import find_neighbors_dist

            def estep():
                c = host_conn.to(dev, non_blocking=True)
                res = find_neighbors_dist(c, et, base, N, p2p=use_p2p)
                outs = []
                for x in (*res.node, *res.elem):   # pinned, async D2H, one sync
                    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
                    h.copy_(x, non_blocking=True)
                    outs.append(h)
                torch.cuda.current_stream().synchronize()
                return outs
        else:
            def estep():
                (no, ni), (eo, ei) = mn.find_neighbors_host(host_conn, et, N, device=dev)
                return [no, ni, eo, ei]

        outs = estep()   # warm the pinned caching allocator
        d2h = sum(x.numel() * x.element_size() for x in outs)
        del outs
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(s)
        for _ in range(args.steps):
            outs = estep()
            del outs
        e1.record(s)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) / args.steps * 1e3
        barrier()
        ems = maxover(max(e0.elapsed_time(e1) / args.steps, wall))
        e2e = {"value": M_total / (ems / 1e3), "unit": "elements/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems, "mode": "one mn_find_neighbors_both_host call per step"}
        if world == 1 and not poly:
            # the stream-of-meshes API (mn_host_pipeline_*): every step still uploads its connectivity
            # and downloads both CSRs, but the upload of step i + 1 overlaps the download of step i
            # (full-duplex PCIe); the K steps are timed from the first submit to the last wait, so
            # the unoverlapped first upload and last download are inside the timed region
            pl = mn.HostPipeline(dev)

            def pipelined(k):
                prev = None
                for _ in range(k):
                    tk = pl.submit(host_conn, et, N)
                    if prev is not None:
                        outs = pl.wait(prev)
                        del outs
                    prev = tk
                return pl.wait(prev)

            outs = pipelined(2)   # warm-up (pinned caching allocator, device pools)
            assert sum(x.numel() * x.element_size() for pair in outs for x in pair) == d2h
            del outs
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            outs = pipelined(args.steps)
            del outs
            pms = (time.perf_counter() - w0) / args.steps * 1e3
            pl.close()
            e2e = {"value": M_total / (pms / 1e3), "unit": "elements/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": pms,
                   "mode": "pipelined (HostPipeline / mn_host_pipeline_*: upload of step i+1 overlaps the download "
                           "of step i; host wall clock from the first submit to the last wait)",
                   "single_call": {"value": M_total / (ems / 1e3), "ms_per_step": ems,
                                   "mode": "one mn_find_neighbors_both_host call per step"}}
        del host_conn

    # ---- CPU baseline: the oracle on a bounded sample, rank 0 at N=1 only ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        T = oracle.host_threads()
        v1, desc1, _, _ = oracle_sample(conn, et, args.cpu_seconds / 2, outputs=args.outputs)
        if poly or T <= 1:
            v, desc, cores = v1, desc1, 1
        else:
            v, desc, _, _ = oracle_sample(conn, et, args.cpu_seconds / 2, outputs=args.outputs, threads=T)
            cores = T
        cpu = {"value": v, "unit": "elements/s", "cores": cores, "kind": "oracle", "sample": desc,
               "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
               "serial": {"value": v1, "cores": 1, "sample": desc1,
                          "note": "the paper's serial baseline (P:L288-290)"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"config {args.config}: {info['desc']}", "elements": M_total, "nodes": N,
                       **({"conn_entries": int(conn[1].numel())} if poly else {}),
                       "parallelism": "single GPU" if world == 1 else
                       f"{world} GPUs: element shards + NCCL all-to-all by owner node range",
                       "l2": "inputs larger than L2 (no flush needed)",
                       "outputs": "node + element CSR" if args.outputs == "both" else
                       "element-sharing node CSR",
                       **({"max_workspace_gb": args.max_workspace_gb, "node_ranges": chunks_used[-1]}
                          if args.max_workspace_gb and not poly and world == 1 else {})},
            "roofline": roofline, "step_roofline": step_roof, "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "parity": parity,
            **({"exchange": exchange} if exchange else {}),
            **({"memory_bound": mem_bound} if mem_bound else {}),
            **({"latency": latency} if latency else {}),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        from paper_1604_04689_b200.dist import release_comms
        release_comms()
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
