"""Calls run under compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the one-CTA
small path (config 1), the staged pipeline with every element path on small meshes (transpose,
LSD onesweep with its decoupled look-back, MSD), the paper-literal node sort (onesweep over u64
keys + the look-back unique/compaction), the look-back scan, polygons, the chunked mode, and a
multi-tile config-2-like sphere.  Each result is checked against the oracle, so a sanitizer-clean
run is also a correct one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import meshgen
import oracle
import paper_1604_04689_b200 as mn


def check(got, exp, what):
    for (go, gi), (eo, ei) in zip(got, exp):
        assert np.array_equal(go.cpu().numpy(), eo) and np.array_equal(gi.cpu().numpy(), ei), what


def main():
    mn.load()
    cases = [("config1_tri_grid_32", meshgen.TRI3, meshgen.tri_grid(32, 32)),
             ("sphere_64x33", meshgen.TRI3, meshgen.uv_sphere(64, 33)),
             ("kuhn_9", meshgen.TET4, meshgen.kuhn_tets(9)),
             ("hex_8_perm", meshgen.HEX8, (meshgen.relabel(*meshgen.hex_grid(8), 3, 4), 729)),
             ("quad_grid_30x40", meshgen.QUAD4, meshgen.quad_grid(30, 40))]
    for name, et, (conn, N) in cases:
        exp = (oracle.node_csr(et, conn, N), oracle.elem_csr(et, conn, N))
        c = conn.cuda()
        for path in ("auto", "radix", "transpose", "msd"):
            mn.set_elem_path(path)
            check(mn.find_neighbors(c, et, N), exp, f"{name} {path}")
        mn.set_elem_path("auto")
        off, idx = mn.find_node_neighbors_sortpairs(c, et, N)
        check([(off, idx)], [exp[0]], f"{name} sortpairs")
        check(mn.find_neighbors_chunked(c, et, N, 1 << 16)[:2], exp, f"{name} chunked")
        print("ok", name, flush=True)
    cnt = torch.randint(0, 50, (100003,), dtype=torch.int32, device="cuda")
    ref = np.concatenate([[0], np.cumsum(cnt.cpu().numpy().astype(np.int64))])
    assert np.array_equal(mn.exclusive_scan(cnt).cpu().numpy(), ref)
    off, idx, N = meshgen.poly_mixed_grid(20, 30, 5)
    got = mn.find_poly_neighbors(off.cuda(), idx.cuda(), N, node=True, elem=True, shared=True)
    check(got, (oracle.poly_node_csr(off, idx, N), oracle.poly_elem_csr(off, idx, N),
                oracle.poly_shared_csr(off, idx, N)), "poly")
    # the pipelined host API: three streams, readbacks through k_read_words, two meshes in flight
    pl = mn.HostPipeline()
    tks = [(pl.submit(conn.contiguous().pin_memory(), et, N), et, conn, N) for _, et, (conn, N) in cases[:3]]
    for tk, et, conn, N in tks:
        node, elem = pl.wait(tk)
        for (go, gi), (eo, ei) in zip((node, elem), (oracle.node_csr(et, conn, N), oracle.elem_csr(et, conn, N))):
            assert np.array_equal(go.numpy(), eo) and np.array_equal(gi.numpy(), ei), "pipeline"
    pl.close()
    print("ok pipeline", flush=True)
    print("ok all", flush=True)


if __name__ == "__main__":
    main()
