"""Diagnostics: run each row on a few meshes and print where the CUDA path first departs from the
oracle (developer tool; not part of the product)."""
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
import oracle  # noqa: E402
from oracle import stages  # noqa: E402
import paper_1604_04689_b200 as mn  # noqa: E402


def unpack(keys, N):
    b = mn.node_key_bits(N)
    k = keys.cpu().numpy()
    k = k.view(np.uint32).astype(np.uint64) if k.dtype == np.int32 else k.view(np.uint64)
    return (k >> np.uint64(b)).astype(np.int64), (k & np.uint64((1 << b) - 1)).astype(np.int64)


def first_diff(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    d = np.nonzero(a != b)[0]
    return "equal" if d.size == 0 else f"{d.size} diffs, first at {d[:5]} got {a[d[:5]]} exp {b[d[:5]]}"


def run(name, et, conn, N):
    print(f"=== {name}: M={conn.shape[0]} N={N} b={mn.node_key_bits(N)} keybytes={mn.node_key_bytes(N)}")
    c = conn.cuda()
    for label, fn in [
        ("a1 emit", lambda: (unpack(mn.emit_node_pairs(c, et, N), N), stages.expand_node_pairs(et, conn))),
        ("a2 emit", lambda: ((lambda k, v: (k.cpu().numpy(), v.cpu().numpy()))(*mn.emit_elem_pairs(c, et, N)),
                             stages.expand_elem_pairs(et, conn))),
        ("a3 sort", lambda: ((lambda k: unpack(mn.radix_sort_keys(k, 2 * mn.node_key_bits(N)), N))(mn.emit_node_pairs(c, et, N)),
                             stages.sort_pairs(*stages.expand_node_pairs(et, conn)))),
        ("whole node", lambda: (tuple(x.cpu().numpy() for x in mn.find_node_neighbors(c, et, N)), oracle.node_csr(et, conn, N))),
        ("whole elem", lambda: (tuple(x.cpu().numpy() for x in mn.find_elem_neighbors(c, et, N)), oracle.elem_csr(et, conn, N))),
    ]:
        try:
            got, exp = fn()
            print(f"  {label}: {first_diff(got[0], exp[0])} | {first_diff(got[1], exp[1])}")
        except Exception as e:  # noqa: BLE001
            print(f"  {label}: EXC {e}")
            traceback.print_exc(limit=2)


if __name__ == "__main__":
    run("single_tri", 0, torch.tensor([[0, 1, 2]], dtype=torch.int32), 3)
    run("two_tri", 0, torch.tensor([[0, 1, 2], [0, 2, 3]], dtype=torch.int32), 4)
    run("tri_grid_2", 0, *meshgen.tri_grid(2, 2))
    run("tri_grid_32", 0, *meshgen.tri_grid(32, 32))
    run("kuhn_3", 2, *meshgen.kuhn_tets(3))
    run("kuhn_10", 2, *meshgen.kuhn_tets(10))
    run("sphere_200", 0, *meshgen.uv_sphere(200, 101))
