"""On-device mesh build (csrc/mesh_build.cu): the fan-CSR built on the
GPU from the uploaded faces equals the host build (itself checked against the reference's
for_each_incident_triangle order in test_capi_host.py) on every golden and synthetic mesh,
and a rejected mesh reports the reference's error text."""

import numpy as np
import pytest

from conftest import FPS_CASES, PTP_CASES, golden
from test_gpu_parity import SYNTH, polar_arrays

import paper_1810_08218_b200 as g

pytestmark = pytest.mark.gpu


def meshes():
    for name in sorted(set(PTP_CASES) | set(FPS_CASES)):
        gd = golden(name)
        yield name, gd["vertices"], gd["faces"]
    for name, make, _ in SYNTH:
        v, f = make()
        yield name, v, f
    v, f = g.grid_arrays(7, 5)
    yield "grid7x5", v, f
    # an isolated vertex (no incident face) and a second component
    v, f = g.icosphere_arrays(2)
    v2 = np.vstack([v, [[5.0, 5.0, 5.0]], v + 3.0])
    f2 = np.vstack([f, f + len(v) + 1])
    yield "two_spheres_isolated", v2, f2.astype(np.int32)
    yield "one_triangle", np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), np.array([[0, 1, 2]],
                                                                                          np.int32)


@pytest.mark.parametrize("name,v,f", list(meshes()), ids=lambda x: x if isinstance(x, str) else "")
def test_device_fans_equal_host_build(name, v, f, monkeypatch):
    monkeypatch.delenv("GEODIST_HOST_BUILD", raising=False)
    cptr, ring, deg = g.build_fans(v, f)
    M = g.Mesh(v, f)
    dc, dr, dd = M.fans()
    assert np.array_equal(dc, cptr)
    assert np.array_equal(dr, ring)
    assert np.array_equal(dd, deg)
    # per-vertex queries read the same (downloaded) arrays
    x = len(v) // 2
    a, b = M.fan(x)
    d = cptr[x + 1] - cptr[x]
    assert np.array_equal(a, ring[cptr[x] + x:cptr[x] + x + d])
    assert np.array_equal(b, ring[cptr[x] + x + 1:cptr[x] + x + d + 1])


def test_device_and_host_build_give_the_same_fields(monkeypatch):
    v, f = polar_arrays(40, 12)
    monkeypatch.setenv("GEODIST_HOST_BUILD", "1")
    a = g.geodesics(g.Mesh(v, f), [0, 200], precision="single", labels=True)
    monkeypatch.delenv("GEODIST_HOST_BUILD")
    b = g.geodesics(g.Mesh(v, f), [0, 200], precision="single", labels=True)
    assert np.array_equal(a["distances"], b["distances"])
    assert np.array_equal(a["labels"], b["labels"])


BAD = [
    ("out of range", np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), [[0, 1, 7]]),
    ("out of range", np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), [[0, 1, 2], [-1, 1, 2]]),
    ("repeats a vertex", np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), [[0, 1, 1]]),
    ("zero-length edge", np.array([[0, 0, 0], [0, 0, 0], [0, 1, 0]], float), [[0, 1, 2]]),
    ("non-finite", np.array([[0, 0, np.nan], [1, 0, 0], [0, 1, 0]]), [[0, 1, 2]]),
    ("non-finite", np.array([[0, 0, 0], [1, np.inf, 0], [0, 1, 0]]), [[0, 1, 2]]),
    ("non-manifold edge", np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float),
     [[0, 1, 2], [0, 1, 2]]),
    ("non-manifold vertex 0",
     np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0]], float),
     [[0, 1, 2], [0, 3, 4]]),
]


@pytest.mark.parametrize("match,v,f", BAD, ids=[b[0] for b in BAD])
def test_device_build_rejects_like_the_reference(match, v, f, monkeypatch):
    monkeypatch.delenv("GEODIST_HOST_BUILD", raising=False)
    f = np.array(f, np.int32)
    with pytest.raises(RuntimeError) as host:
        g.build_fans(v, f)
    with pytest.raises(RuntimeError, match=match) as dev:
        g.Mesh(v, f)
    assert str(dev.value) == str(host.value)


def test_large_mesh_device_build_matches_host():
    v, f = g.torus_arrays(700, 500)
    cptr, ring, deg = g.build_fans(v, f)
    dc, dr, dd = g.Mesh(v, f).fans()
    assert np.array_equal(dc, cptr) and np.array_equal(dr, ring) and np.array_equal(dd, deg)
