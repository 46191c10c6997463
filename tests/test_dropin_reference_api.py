"""GPU: the reference's OWN code running on the B200 backend.

integration/Makefile rebuilds, against the C++ drop-in (integration/cpp/
geodist_b200_dropin.cpp over include/geodist_b200.h), two unmodified reference
artefacts: the acceptance suite (proj/tests/acceptance.cpp) and the pybind11
module (proj/python/bindings.cpp).  Their outputs must equal the reference
library's: the acceptance report line for line (tests/golden/
acceptance_reference.txt, timings stripped) and the distance fields bit for bit
(tests/golden/*.npz)."""

import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import FPS_CASES, PTP_CASES, ROOT, bits, golden

pytestmark = pytest.mark.gpu
BUILD = os.path.join(ROOT, "integration", "_build")


def _need(path):
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run make -C integration (needs /root/reference at build time)")


def test_reference_acceptance_suite_on_b200():
    exe = os.path.join(BUILD, "acceptance")
    _need(exe)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600).stdout
    got = [re.sub(r" \[[0-9.]+s\]$", "", ln) for ln in out.splitlines()]
    want = open(os.path.join(ROOT, "tests", "golden", "acceptance_reference.txt")).read().splitlines()
    assert got == want


@pytest.fixture(scope="module")
def refmod():
    _need(os.path.join(BUILD, "geodist"))
    sys.path.insert(0, BUILD)
    import geodist
    assert geodist.__file__.startswith(BUILD)
    return geodist


@pytest.mark.parametrize("name", PTP_CASES)
def test_reference_bindings_geodesics(refmod, name):
    gd = golden(name)
    mesh = refmod.mesh_from_arrays(gd["vertices"], gd["faces"])
    labels = "labels_d" in gd
    for p, prec in (("s", "single"), ("d", "double")):
        r = refmod.geodesics(mesh, gd["sources"].tolist(), precision=prec, labels=labels)
        assert np.array_equal(bits(r["distances"]), bits(gd[f"dist_{p}"]))
        assert r["iterations"] == int(gd[f"K_{p}"])
        assert r["relax_calls"] == int(gd[f"relax_{p}"])
        if labels:
            assert np.array_equal(r["labels"], gd[f"labels_{p}"])
    t = refmod.toplesets(mesh, gd["sources"].tolist())
    assert np.array_equal(t["sorted"], gd["sorted"]) and np.array_equal(t["limits"], gd["limits"])


@pytest.mark.parametrize("name", FPS_CASES)
def test_reference_bindings_fps_voronoi(refmod, name):
    gd = golden(name)
    mesh = refmod.mesh_from_arrays(gd["vertices"], gd["faces"])
    r = refmod.farthest_point_sampling(mesh, int(gd["m"]), seed=int(gd["seed"]))
    assert np.array_equal(r["samples"], gd["samples_d"])
    assert np.array_equal(r["labels"], gd["labels_d"])
    assert r["radius"] == float(gd["radius_d"])
    assert [h["relax_calls"] for h in r["history"]] == list(gd["hist_relax_d"])
    lab = refmod.voronoi(mesh, gd["samples_d"].tolist())
    assert np.array_equal(lab, gd["voronoi_d"])


def test_reference_smoke_assertions(refmod):
    # the assertions of the reference's tests/python/test_smoke.py on the B200 backend
    g = refmod
    grid = g.generate_grid(5, 4)
    assert grid.n_vertices == 20 and grid.n_faces == 24
    assert g.generate_icosphere(0).degree_histogram() == {5: 12}
    with pytest.raises(RuntimeError):
        g.mesh_from_arrays(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float),
                           np.array([[0, 1, 7]], np.int32))
    mesh = g.generate_grid(9, 9)
    exact = g.grid_reference(mesh, [0])
    ptp = g.geodesics(mesh, [0], method="ptp")
    dij = g.geodesics(mesh, [0], method="dijkstra")
    assert np.all(ptp["distances"] >= exact * (1 - 1e-12))
    assert np.all(ptp["distances"] <= dij["distances"] + 1e-15)
    mesh = g.generate_grid(41, 41)
    c = 20 * 41 + 20
    rep = g.mape(g.geodesics(mesh, [c])["distances"], g.grid_reference(mesh, [c]), [c])
    assert rep["mape"] < 3.5
    levels = g.toplesets(g.generate_grid(7, 7), [24])
    assert sorted(levels["sorted"].tolist()) == list(range(49))
    mesh = g.generate_grid(21, 21, 2.0)
    one = g.geodesics(mesh, [0, 440], workers=1)
    many = g.geodesics(mesh, [0, 440], workers=8)
    assert np.array_equal(one["distances"], many["distances"])
