"""CPU: the C-ABI library loads, exports every symbol include/geodist_b200.h
declares, and its host logic (validation, rotational fans, generators) matches
the reference; compute entry points fail loudly without an sm_100 GPU."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

import paper_1810_08218_b200 as g
from paper_1810_08218_b200 import _capi


def header_symbols():
    text = open(os.path.join(ROOT, "include", "geodist_b200.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(geodist_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    L = _capi.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    assert sorted(_capi.EXPORTED) == syms
    for s in syms:
        assert hasattr(L, s), s
    assert L.geodist_version() >= 100


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_capi.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.parametrize("name", ["ico3_src0", "ico2_src0", "grid33_shear2_two", "grid9x5_corners"])
def test_generators_bit_identical_to_reference(name):
    gd = golden(name)
    n = len(gd["vertices"])
    if name.startswith("ico"):
        sub = {642: 3, 162: 2}[n]
        v, f = g.icosphere_arrays(sub)
    else:
        nx, ny, sh = {"grid33_shear2_two": (33, 33, 2.0), "grid9x5_corners": (9, 5, 0.0)}[name]
        v, f = g.grid_arrays(nx, ny, sh)
    assert np.array_equal(v.view(np.int64), gd["vertices"].view(np.int64))
    assert np.array_equal(f, gd["faces"])


def test_fans_match_reference_order():
    from oracle import ref
    from oracle import port
    meshes = [g.icosphere_arrays(3), g.grid_arrays(9, 7, 2.0), g.torus_arrays(12, 9)]
    for v, f in meshes:
        cptr, ring, deg = g.build_fans(v, f)
        P = port.PortMesh(v, f)
        R = ref.RefMesh.from_arrays(v, f) if ref.available() else None
        for x in range(len(v)):
            d = cptr[x + 1] - cptr[x]
            r0 = cptr[x] + x
            v1 = ring[r0:r0 + d]
            v2 = ring[r0 + 1:r0 + d + 1]
            a, b, extra = P.fan(x)
            assert np.array_equal(v1, a) and np.array_equal(v2, b)
            assert deg[x] == (d + 1 if extra >= 0 else d)
            if R is not None:
                ra, rb, rextra = R.fan(x)
                assert np.array_equal(ra, a) and np.array_equal(rb, b) and rextra == extra


def test_validation_messages():
    tri = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    with pytest.raises(RuntimeError, match="out of range"):
        g.build_fans(tri, np.array([[0, 1, 7]]))
    with pytest.raises(RuntimeError, match="repeats a vertex"):
        g.build_fans(tri, np.array([[0, 1, 1]]))
    with pytest.raises(RuntimeError, match="zero-length edge"):
        g.build_fans(np.array([[0, 0, 0], [0, 0, 0], [0, 1, 0]], float), np.array([[0, 1, 2]]))
    with pytest.raises(RuntimeError, match="non-finite"):
        g.build_fans(np.array([[0, 0, np.nan], [1, 0, 0], [0, 1, 0]]), np.array([[0, 1, 2]]))
    with pytest.raises(RuntimeError, match="non-manifold edge"):
        g.build_fans(tri, np.array([[0, 1, 2], [0, 1, 2]]))
    # bowtie: two fans meeting at vertex 0
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0]], float)
    with pytest.raises(RuntimeError, match="non-manifold vertex 0"):
        g.build_fans(v, np.array([[0, 1, 2], [0, 3, 4]]))
    with pytest.raises(RuntimeError):
        g.mesh_from_arrays(tri, np.array([[0, 1, 7]], np.int32))
    with pytest.raises(ValueError):
        g.mesh_from_arrays(tri[:, :2], np.array([[0, 1, 2]]))


def test_synthetic_generators():
    v, f = g.torus_arrays(40, 30)
    assert v.shape == (1200, 3) and f.shape == (2400, 3)
    cptr, ring, deg = g.build_fans(v, f)
    assert set(np.unique(deg)) == {6}  # closed torus, every vertex valence 6
    a, _ = g.noisy_icosphere_arrays(3, 2e-3, 1)
    b, _ = g.noisy_icosphere_arrays(3, 2e-3, 1)
    c, _ = g.icosphere_arrays(3)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    r = np.linalg.norm(a, axis=1)
    assert 0.99 < r.min() and r.max() < 1.01
    h, _ = g.heightfield_arrays(64, 64)
    assert np.allclose(h[:, 2], 20 * np.sin(h[:, 0] / 97) * np.cos(h[:, 1] / 131))


def test_compute_fails_loudly_without_gpu():
    if g.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="CUDA"):
        g.generate_icosphere(1)


@pytest.mark.parametrize("kind", ["torus", "noisy_icosphere", "heightfield"])
def test_synthetic_generators_equal_reference_side_generators(kind):
    """The bench's reference arm builds its meshes with oracle/ref_capi.cpp's generators
    (reference types, no product library): they must give the product's arrays bit for bit."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    if kind == "torus":
        R, (v, f) = ref.RefMesh.torus(57, 31), g.torus_arrays(57, 31)
    elif kind == "noisy_icosphere":
        R, (v, f) = ref.RefMesh.noisy_icosphere(4, 2e-3, 1), g.noisy_icosphere_arrays(4, 2e-3, 1)
    else:
        R, (v, f) = ref.RefMesh.heightfield(65, 33), g.heightfield_arrays(65, 33)
    rv, rf = R.arrays()
    assert np.array_equal(rv.view(np.int64), v.view(np.int64))
    assert np.array_equal(rf, f)


def test_source_index_beyond_int32_rejected():
    """an int64 source index must not wrap onto another vertex."""
    with pytest.raises(ValueError, match="out of range"):
        g._sources([2 ** 32])
    with pytest.raises(ValueError, match="out of range"):
        g._sources([0, -2 ** 40])
    assert g._sources([5, 7]).dtype == np.int32
