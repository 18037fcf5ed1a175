"""Native OFF / OBJ ingestion (mn_parse_off / mn_parse_obj; SPEC.md mesh-io,
S:L111-146).  Host code: these tests run without a GPU."""
import numpy as np
import pytest

import meshgen

mn = pytest.importorskip("paper_1604_04689_b200")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1604_04689_b200 import build
    build.build()


def _off(text):
    return mn.load_off(text.encode() if isinstance(text, str) else text)


def _obj(text):
    return mn.load_obj(text.encode() if isinstance(text, str) else text)


def _rings(off, idx):
    off, idx = off.numpy(), idx.numpy()
    return [idx[off[e]:off[e + 1]].tolist() for e in range(len(off) - 1)]


def _err(fn, data):
    with pytest.raises(mn.MeshError) as ei:
        fn(data)
    return ei.value.code, ei.value.elem, ei.value.pos


# ---- SPEC examples ------------------------------------------------------------
def test_spec_off_minimal():                      # S:L124 "minimal OFF"
    off, idx, N, k = _off("OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n")
    assert (N, k, _rings(off, idx)) == (3, 3, [[0, 1, 2]])


def test_spec_off_out_of_range():                 # S:L125 "index 5 >= 3"
    assert _err(_off, "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 5\n") == (mn.MN_ERR_INDEX_OUT_OF_RANGE, 0, 2)


def test_spec_obj_one_based():
    off, idx, N, _ = _obj("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    assert (N, _rings(off, idx)) == (3, [[0, 1, 2]])


def test_spec_obj_suffixes():                     # S:L134 "f 1/1/1 2/2/2 3/3/3"
    off, idx, N, _ = _obj("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1/1/1 2/2/2 3/3/3\nf 1//1 2/2 3\n")
    assert _rings(off, idx) == [[0, 1, 2], [0, 1, 2]]


def test_spec_obj_negative():                     # S:L135 "f -3 -2 -1 after 3 vertices"
    off, idx, N, _ = _obj("v 0 0 0\nv 1 0 0\nv 0 1 0\nf -3 -2 -1\nv 2 2 2\nf -4 -1 -2\n")
    assert (N, _rings(off, idx)) == (4, [[0, 1, 2], [0, 3, 2]])


def test_spec_obj_zero_index():                   # S:L131 "ZeroIndex (OBJ index 0 is invalid)"
    assert _err(_obj, "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 0 3\n") == (mn.MN_ERR_ZERO_INDEX, 4, 2)


# ---- format rules (R19) ------------------------------------------------------------
def test_off_header_variants_comments_crlf_tabs():
    a = _off("OFF 4 2 5\r\n# comment\r\n0 0 0\r\n1 0 0\r\n\r\n1 1 0\r\n0 1 0\r\n3\t0 1 2\r\n3 0  2 3 255 0 0\r\n")
    b = _off("4 2 0\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n3 0 1 2\n3 0 2 3\n")
    assert _rings(a[0], a[1]) == _rings(b[0], b[1]) == [[0, 1, 2], [0, 2, 3]]
    assert a[2] == b[2] == 4


def test_polygons_kept():                         # S:L143 "arity > 3 kept as Polygon"
    off, idx, N, k = _obj("v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nv 2 0 0\nf 1 2 3 4\nf 2 5 3\n")
    assert k == 0 and _rings(off, idx) == [[0, 1, 2, 3], [1, 4, 2]]
    off, idx, N, k = _off("OFF\n4 1 0\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n4 0 1 2 3\n")
    assert k == 4


def test_obj_ignores_other_records():
    off, idx, N, _ = _obj("# c\nmtllib a.mtl\no obj\nv 0 0 0\nvt 0 0\nvn 0 0 1\nv 1 0 0 1.0\nv 0 1 0\n"
                                 "g grp\nusemtl m\ns off\nl 1 2\nf 1 2 3\n")
    assert (N, _rings(off, idx)) == (3, [[0, 1, 2]])


@pytest.mark.parametrize("data,code,line", [
    ("OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n", mn.MN_ERR_COUNT_MISMATCH, 5),           # missing face line
    ("OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n3 0 1 2\n", mn.MN_ERR_COUNT_MISMATCH, 7),   # extra content
    ("OFF\n3 x 0\n", mn.MN_ERR_SYNTAX, 2),
    ("OFF\n3 1 0\n0 0 0\n1 zero 0\n0 1 0\n3 0 1 2\n", mn.MN_ERR_SYNTAX, 4),
    ("OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1\n", mn.MN_ERR_SYNTAX, 6),              # k says 3, 2 given
    ("OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2.5\n", mn.MN_ERR_SYNTAX, 6),
    ("", mn.MN_ERR_COUNT_MISMATCH, 0),
])
def test_off_errors(data, code, line):
    c, e, _ = _err(_off, data)
    assert (c, e) == (code, line)


@pytest.mark.parametrize("data,code,elem,pos", [
    ("v 0 0\n", mn.MN_ERR_SYNTAX, 1, 3),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 x\n", mn.MN_ERR_SYNTAX, 4, 3),
    ("v 0 0 0\nv 1 0 0\nf 1 2\n", mn.MN_ERR_ARITY, 0, -1),                       # validation: (face, pos)
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 2\n", mn.MN_ERR_DEGENERATE, 0, 2),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 -4\n", mn.MN_ERR_INDEX_OUT_OF_RANGE, 0, 2),
])
def test_obj_errors(data, code, elem, pos):
    assert _err(_obj, data) == (code, elem, pos)


def test_path_argument(tmp_path):
    p = tmp_path / "m.obj"
    p.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    off, idx, N, _ = mn.load_obj(str(p))
    assert _rings(off, idx) == [[0, 1, 2]]


def test_str_text_and_pathlike(tmp_path):
    """A str holding the file's text is parsed as text; os.PathLike and line-free str are paths."""
    off, idx, N, _ = mn.load_obj("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    assert _rings(off, idx) == [[0, 1, 2]] and N == 3
    p = tmp_path / "m.off"
    p.write_text("OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n")
    assert _rings(*mn.load_off(p)[:2]) == [[0, 1, 2]]


def test_untrusted_face_count_is_not_reserved():
    """A header claiming 2^31-1 faces in a 40-byte file is a count mismatch, not an allocation of
    16 GB (no C++ exception escapes the C ABI)."""
    assert _err(_off, "OFF\n3 2147483647 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n")[0] == mn.MN_ERR_COUNT_MISMATCH


def test_empty_obj_and_off():
    off, idx, N, k = _obj("")
    assert off.tolist() == [0] and idx.numel() == 0 and N == 0
    off, idx, N, k = _off("OFF\n2 0 0\n0 0 0\n1 1 1\n")
    assert off.tolist() == [0] and N == 2


# ---- round trips of generated meshes --------------------------------------------------------
def _to_off(off, idx, N):
    off, idx = off.numpy(), idx.numpy()
    lines = ["OFF", f"{N} {len(off) - 1} 0"] + [f"{v % 7}.5 {v % 3} -{v}" for v in range(N)]
    lines += [" ".join(map(str, [off[e + 1] - off[e], *idx[off[e]:off[e + 1]]])) for e in range(len(off) - 1)]
    return "\n".join(lines) + "\n"


def _to_obj(off, idx, N, negative=False):
    off, idx = off.numpy(), idx.numpy()
    lines = [f"v {v} 0 {v % 5}" for v in range(N)]
    for e in range(len(off) - 1):
        ring = idx[off[e]:off[e + 1]]
        toks = [str(int(x) - N) if negative else f"{int(x) + 1}/{e}/{e}" for x in ring]
        lines.append("f " + " ".join(toks))
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("make", [lambda: (*meshgen.poly_from_conn(meshgen.tri_grid(9, 7)[0]), 80),
                                  lambda: meshgen.poly_mixed_grid(12, 10, 3), lambda: meshgen.honeycomb(6, 5),
                                  lambda: meshgen.random_poly(300, 90, 3, 9, 1)])
def test_round_trip(make):
    off, idx, N = make()
    for text, fn in ((_to_off(off, idx, N), _off), (_to_obj(off, idx, N), _obj),
                     (_to_obj(off, idx, N, negative=True), _obj)):
        o2, i2, n2, k = fn(text)
        assert n2 == N and np.array_equal(o2.numpy(), off.numpy()) and np.array_equal(i2.numpy(), idx.numpy())
        # mesh stats: the face count equals an independent count of face lines
        nf = sum(1 for ln in text.splitlines() if ln.startswith("f ")) if fn is _obj else \
            int(text.splitlines()[1].split()[1])
        assert o2.numel() - 1 == nf


def test_fuzz_never_crashes():
    """Random byte mutations of valid files: always a typed status, never a crash or a mesh that
    violates the invariants."""
    off, idx, N = meshgen.poly_mixed_grid(5, 4, 2)
    rng = np.random.default_rng(0)
    for base, fn in ((_to_off(off, idx, N), _off), (_to_obj(off, idx, N), _obj)):
        raw = bytearray(base.encode())
        for trial in range(400):
            b = bytearray(raw)
            for _ in range(int(rng.integers(1, 6))):
                op = rng.integers(0, 3)
                p = int(rng.integers(0, len(b)))
                if op == 0:
                    b[p] = int(rng.choice(list(b"0123456789 -/\n\t#fvOFx.\r")))
                elif op == 1:
                    del b[p]
                else:
                    b.insert(p, int(rng.integers(0, 256)))
            try:
                o, i, n, _ = fn(bytes(b))
            except mn.MeshError as e:
                assert e.code in (mn.MN_ERR_SYNTAX, mn.MN_ERR_COUNT_MISMATCH, mn.MN_ERR_ZERO_INDEX, mn.MN_ERR_ARITY,
                                  mn.MN_ERR_INDEX_OUT_OF_RANGE, mn.MN_ERR_DEGENERATE, mn.MN_ERR_CAPACITY)
                continue
            o, i = o.numpy(), i.numpy()
            assert o[0] == 0 and o[-1] == len(i) and (np.diff(o) >= 3).all()
            assert ((i >= 0) & (i < n)).all()
