"""Diagnostics for the element-CSR node path: print nodes whose neighbour list differs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
import oracle  # noqa: E402
import paper_1604_04689_b200 as mn  # noqa: E402

for n in (2, 3, 10):
    conn, N = meshgen.kuhn_tets(n)
    (no, ni), (eo, ei) = mn.find_neighbors(conn.cuda(), "tet4", N)
    no, ni, eo, ei = (x.cpu().numpy() for x in (no, ni, eo, ei))
    ro, ri = oracle.node_csr(2, conn, N)
    so, si = oracle.elem_csr(2, conn, N)
    print(f"kuhn {n}: elem ok={np.array_equal(eo, so) and np.array_equal(ei, si)} "
          f"node off ok={np.array_equal(no, ro)} idx ok={np.array_equal(ni, ri)}")
    bad = 0
    for v in range(N):
        g, e = ni[no[v]:no[v + 1]], ri[ro[v]:ro[v + 1]]
        if not np.array_equal(g, e):
            bad += 1
            if bad <= 6:
                print(f"  node {v} deg {so[v+1]-so[v]} got {g.tolist()} exp {e.tolist()}")
    print("  bad nodes", bad)
    # node-only call
    o2, i2 = mn.find_node_neighbors(conn.cuda(), "tet4", N)
    print("  node-only idx ok", np.array_equal(i2.cpu().numpy(), ri))
