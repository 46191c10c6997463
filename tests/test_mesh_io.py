"""Mesh files (csrc/mesh_io.cpp) against the reference's own
load_mesh / write_mesh (src/mesh_io.cpp, built into oracle/_ref): identical arrays,
identical bytes written, identical error messages.  Host-only."""

import numpy as np
import pytest

import paper_1810_08218_b200 as g
from oracle import ref

needs_ref = pytest.mark.skipif(not ref.available(), reason="reference library not built")


def ref_read(path):
    m = ref.RefMesh.load(path)
    return m.arrays()


def both(path):
    """(ours, reference): arrays or the exception text."""
    out = []
    for fn in (g.read_mesh, ref_read):
        try:
            v, f = fn(path)
            out.append((np.asarray(v, np.float64).reshape(-1, 3), np.asarray(f, np.int32).reshape(-1, 3)))
        except (RuntimeError, ValueError) as e:
            out.append(str(e))
    return out


MESHES = {
    "ico2": lambda: g.icosphere_arrays(2),
    "grid_shear": lambda: g.grid_arrays(7, 5, 0.3),
    "noisy_ico3": lambda: g.noisy_icosphere_arrays(3, 2e-3, 1),
    "torus": lambda: g.torus_arrays(16, 11),
}


@pytest.mark.parametrize("name", sorted(MESHES))
@pytest.mark.parametrize("ext", ["off", "obj"])
def test_round_trip_bit_exact(tmp_path, name, ext):
    v, f = MESHES[name]()
    p = tmp_path / f"m.{ext}"
    g.write_mesh(p, v, f)
    rv, rf = g.read_mesh(p)
    assert np.array_equal(rv.view(np.int64), np.asarray(v, np.float64).view(np.int64))
    assert np.array_equal(rf, f)


@needs_ref
@pytest.mark.parametrize("name", sorted(MESHES))
@pytest.mark.parametrize("ext", ["off", "obj"])
def test_writer_bytes_and_reader_match_reference(tmp_path, name, ext):
    v, f = MESHES[name]()
    ours, theirs = tmp_path / f"a.{ext}", tmp_path / f"b.{ext}"
    g.write_mesh(ours, v, f)
    ref.RefMesh.from_arrays(v, f).write(theirs, obj=ext == "obj")
    assert ours.read_bytes() == theirs.read_bytes()
    a, b = both(ours)
    assert np.array_equal(a[0].view(np.int64), b[0].view(np.int64)) and np.array_equal(a[1], b[1])


TRI = "0 0 0\n1 0 0\n0 1 0\n"
CASES = {
    # accepted variants
    "comments.off": "# c\n\nOFF\n# counts next\n3 1 0\n" + TRI + "\n# x\n3 0 1 2\n",
    "inline_counts.off": "OFF 3 1 0\n" + TRI + "3 0 1 2\n",
    "crlf.off": "OFF\r\n3 1 0\r\n0 0 0\r\n1 0 0\r\n0 1 0\r\n3 0 1 2\r\n",
    "signs_exp.off": "OFF\n3 1 0\n+0 -0.0 0e0\n1.5e-1 .25 0\n1. 1E+1 -2.5E-3\n3 0 1 2\n",
    "trailing.off": "OFF\n3 1 0\n0 0 0 extra\n1 0 0 1 1\n0 1 0.5x\n3 0 1 2 9\n",
    "partial_header.off": "OFF 3 1\n3 1 0\n" + TRI + "3 0 1 2\n",
    "slashes.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nvt 0 0\nvn 0 0 1\nf 1/1/1 2//1 3/1\n",
    "negative.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf -3 -2 -1\n",
    "misc.obj": "# c\no thing\nv 0 0 0 1\nv 1 0 0\nusemtl x\nv 0 1 0\ns off\nf 1 2 3\n",
    # errors
    "empty.off": "\n# nothing\n",
    "header.off": "OF\n3 1 0\n" + TRI + "3 0 1 2\n",
    "nocounts.off": "OFF\n",
    "badcounts.off": "OFF\n3 x 0\n",
    "negcounts.off": "OFF\n-3 1 0\n",
    "eof_vertex.off": "OFF\n3 1 0\n0 0 0\n",
    "bad_vertex.off": "OFF\n3 1 0\n0 0 0\n1 x 0\n0 1 0\n3 0 1 2\n",
    "bad_exp.off": "OFF\n3 1 0\n0 0 0\n1 0 1e\n0 1 0\n3 0 1 2\n",
    "inf.off": "OFF\n3 1 0\n0 0 0\n1 0 inf\n0 1 0\n3 0 1 2\n",
    "eof_face.off": "OFF\n3 1 0\n" + TRI,
    "quad.off": "OFF\n4 1 0\n" + TRI + "1 1 0\n4 0 1 2 3\n",
    "bad_face.off": "OFF\n3 1 0\n" + TRI + "3 0 1\n",
    "float_index.off": "OFF\n3 1 0\n" + TRI + "3.0 0 1 2\n",
    "range.off": "OFF\n3 1 0\n" + TRI + "3 0 1 7\n",
    "repeat.off": "OFF\n3 1 0\n" + TRI + "3 0 1 1\n",
    "zero_edge.off": "OFF\n3 1 0\n0 0 0\n0 0 0\n0 1 0\n3 0 1 2\n",
    "bad_v.obj": "v 0 0\n",
    "quad.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\nf 1 2 4 3\n",
    "bad_index.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 a\n",
    "plus_index.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf +1 2 3\n",
    "zero_index.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n",
    "rel_range.obj": "v 0 0 0\nv 1 0 0\nf -3 1 2\n",
    "range.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 9\n",
    "mesh.ply": "ply\n",
}


@needs_ref
@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(tmp_path, name):
    p = tmp_path / name
    p.write_text(CASES[name])
    a, b = both(p)
    if isinstance(b, str):
        assert a == b
    else:
        assert not isinstance(a, str), a
        assert np.array_equal(a[0].view(np.int64), b[0].view(np.int64))
        assert np.array_equal(a[1], b[1])


@needs_ref
def test_missing_file_message(tmp_path):
    a, b = both(tmp_path / "nope.off")
    assert a == b and "cannot open file" in a


def test_reader_errors_without_reference(tmp_path):
    p = tmp_path / "q.off"
    p.write_text(CASES["quad.off"])
    with pytest.raises(RuntimeError, match="only triangles are supported"):
        g.read_mesh(p)
    with pytest.raises(RuntimeError, match="unsupported mesh format"):
        g.read_mesh(tmp_path / "x.stl")


@needs_ref
@pytest.mark.parametrize("ext", ["off", "obj"])
def test_chunked_parse_matches_reference(tmp_path, ext):
    """Files above the chunking threshold (4 MiB): relative OBJ indices resolved across
    chunk boundaries, and the first error in file order wins over later ones."""
    v, f = g.grid_arrays(400, 400, 0.25)  # 10-20 MB: several chunks
    p = tmp_path / f"big.{ext}"
    g.write_mesh(p, v, f)
    if ext == "obj":
        # rewrite every face with relative (negative) indices interleaved after its vertices
        lines = [f"v {float(x[0])!r} {float(x[1])!r} {float(x[2])!r}" for x in v]
        out = []
        k = 0
        for t, tri in enumerate(f):
            need = int(max(tri)) + 1
            while k < need:
                out.append(lines[k])
                k += 1
            out.append("f " + " ".join(str(int(i) - k) for i in tri))
        out += lines[k:]
        p.write_text("\n".join(out) + "\n")
    a, b = both(p)
    assert not isinstance(a, str) and not isinstance(b, str)
    assert np.array_equal(a[0].view(np.int64), b[0].view(np.int64)) and np.array_equal(a[1], b[1])
    text = p.read_text().splitlines()
    n = len(text)
    for early, late in ((n // 5, 4 * n // 5), (4 * n // 5, n - 2)):
        bad = list(text)
        for at in (early, late):
            bad[at] = "v 1 x 2" if ext == "obj" else ("1 x 2" if at < 1 + len(v) + 1 else "4 1 2 3 4")
        q = tmp_path / f"bad.{ext}"
        q.write_text("\n".join(bad) + "\n")
        a, b = both(q)
        assert isinstance(b, str) and a == b
