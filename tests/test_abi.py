"""CPU-only checks of the boundary: libmeshnbr.so builds for sm_100a, loads, and exports every
symbol include/meshnbr.h declares; host-only entry points answer without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1604_04689_b200 import build as mnbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "meshnbr.h")


@pytest.fixture(scope="module")
def lib():
    path = mnbuild.build()
    return ctypes.CDLL(path)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(mn_[a-z0-9_]+)\s*\(", src)
    return sorted(set(n for n in names if not n.endswith("_t")))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("mn_find_node_neighbors", "mn_find_elem_neighbors", "mn_find_neighbors_both",
                     "mn_find_neighbors_both_host", "mn_csr_release", "mn_radix_sort_keys",
                     "mn_unique_node_csr", "mn_exclusive_scan_i32", "mn_dist_bucket", "mn_dist_finish"):
        assert required in names


def test_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_dynamic_symbol_table_matches_header():
    out = subprocess.run(["nm", "-D", "--defined-only", mnbuild.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mn_[a-z0-9_]+)$", out, flags=re.M))
    assert set(declared_functions()) <= exported


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", mnbuild.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points(lib):
    import paper_1604_04689_b200 as mn
    assert mn.load().mn_abi_version() == 1
    assert mn.load().mn_status_string(2) == b"node index out of range"
    # b = max(1, bit_length(N-1)) (R11)
    assert [mn.node_key_bits(n) for n in (0, 1, 2, 3, 4, 5, 1089, 2 ** 20, 2 ** 20 + 1)] == \
        [1, 1, 1, 2, 2, 3, 11, 20, 21]
    assert mn.node_key_bytes(1089) == 4 and mn.node_key_bytes(501002) == 8
    assert mn.node_key_bytes(65536) == 4 and mn.node_key_bytes(65537) == 8
    # workspace estimate, config 3 both modes: 4 element-pair buffers of 4 B per incidence at least
    Pe = 4 * 12582912
    ws = mn.workspace_bytes("tet4", 12582912, 2146689, 3)
    assert 16 * Pe <= ws < 24 * Pe
    # chunked mode: the per-range estimate shrinks with the number of ranges
    w = [mn.chunk_workspace_bytes("tet4", 12582912, 2146689, k) for k in (1, 2, 4, 8)]
    assert all(a > b for a, b in zip(w, w[1:])) and w[0] < ws
    with pytest.raises(mn.MeshError):
        mn.workspace_bytes("tet4", -1, 10, 3)


def test_no_cpu_fallback_without_device():
    import torch

    import paper_1604_04689_b200 as mn
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(TypeError):
        mn.find_node_neighbors(torch.zeros((1, 3), dtype=torch.int32), "tri3", 3)
