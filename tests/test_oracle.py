"""CPU: the C restatement (oracle/ptp_oracle.c) against the reference's golden
vectors (tests/golden, generated from the unmodified reference by
oracle/gen_golden.py) and its known-answer tests, plus a live cross-check
against the reference build (oracle/_ref) when it is present."""

import math

import numpy as np
import pytest

from conftest import FPS_CASES, PTP_CASES, bits, golden


@pytest.mark.parametrize("name", PTP_CASES)
def test_port_matches_golden(port_lib, name):
    g = golden(name)
    P = port_lib.PortMesh(g["vertices"], g["faces"])
    src = g["sources"]
    t = P.toplesets(src)
    assert np.array_equal(t["sorted"], g["sorted"])
    assert np.array_equal(t["limits"], g["limits"])
    assert np.array_equal(t["position"], g["position"])
    assert t["unreached"] == int(g["unreached"])
    labels = "labels_d" in g
    for p, prec in (("s", "single"), ("d", "double")):
        r = P.ptp(src, precision=prec, labels=labels, trace=True)
        assert np.array_equal(bits(r["distances"]), bits(g[f"dist_{p}"])), prec
        assert r["iterations"] == int(g[f"K_{p}"])
        assert r["relax_calls"] == int(g[f"relax_{p}"])
        assert r["degenerate_calls"] == int(g[f"degen_{p}"])
        assert np.array_equal(r["trace"]["kijU"], g[f"trace_kijU_{p}"])
        assert np.array_equal(bits(r["trace"]["max_rel"]), bits(g[f"trace_maxrel_{p}"]))
        assert np.array_equal(r["trace"]["converged"], g[f"trace_conv_{p}"])
        assert np.array_equal(r["last_change"], g[f"last_change_{p}"])
        if labels:
            assert np.array_equal(r["labels"], g[f"labels_{p}"])


@pytest.mark.parametrize("name", FPS_CASES)
def test_port_fps_matches_golden(port_lib, name):
    g = golden(name)
    P = port_lib.PortMesh(g["vertices"], g["faces"])
    for p, prec in (("s", "single"), ("d", "double")):
        r = P.fps(int(g["m"]), int(g["seed"]), precision=prec)
        assert np.array_equal(r["samples"], g[f"samples_{p}"])
        assert np.array_equal(r["labels"], g[f"labels_{p}"])
        assert r["radius"] == float(g[f"radius_{p}"])
        assert [h["rho"] for h in r["history"]] == list(g[f"hist_rho_{p}"])
        assert [h["relax_calls"] for h in r["history"]] == list(g[f"hist_relax_{p}"])


def test_port_planar_matches_golden(port_lib):
    g = golden("planar_update")
    for p, single in (("s", True), ("d", False)):
        for q in range(len(g["t1"])):
            v, s, d = port_lib.planar(g["x1"][q], g["x2"][q], g["t1"][q], g["t2"][q], single)
            assert bits([v])[0] == bits([g[f"value_{p}"][q]])[0], q
            assert s == g[f"side_{p}"][q] and d == g[f"degen_{p}"][q]


def test_planar_known_answers(port_lib):
    # test_update_kernel.cpp:17-52
    v, s, d = port_lib.planar([1, 0, 0], [0.5, math.sqrt(3) / 2, 0], 0, 0)
    assert abs(v - math.sqrt(3) / 2) <= 1e-15 and not d
    assert port_lib.planar([1, 0, 0], [0.3, 0.9, 0], 0, math.inf)[:2] == (1.0, 0)
    assert port_lib.planar([1, 0, 0], [0, 1, 0], math.inf, math.inf)[:2] == (math.inf, -1)
    assert port_lib.planar([0, -1, 0], [1, -1, 0], 0, 1)[:2] == (1.0, 0)
    v, s, d = port_lib.planar([1, 0, 0], [2, 0, 0], 0.1, 0.2)
    assert d and abs(v - 1.1) < 1e-15


def test_single_triangle(port_lib):
    # test_ptp.cpp:33-42, test_toplesets.cpp:46-52
    P = port_lib.PortMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    t = P.toplesets([0])
    assert list(t["sorted"]) == [0, 1, 2] and list(t["limits"]) == [0, 1, 3]
    r = P.ptp([0], trace=True)
    assert list(r["distances"]) == [0.0, 1.0, 1.0] and r["iterations"] <= 3


def test_errors(port_lib):
    P = port_lib.PortMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    with pytest.raises(ValueError):
        P.toplesets([])
    with pytest.raises(ValueError):
        P.toplesets([7])
    with pytest.raises(ValueError):
        P.toplesets([1, 1])
    with pytest.raises(ValueError):
        P.ptp([0], epsilon=0.0)
    with pytest.raises(RuntimeError):
        port_lib.PortMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 7]])


def test_port_vs_live_reference(port_lib):
    from oracle import ref
    if not ref.available():
        pytest.skip("reference build (oracle/_ref) not present")
    for R in (ref.RefMesh.icosphere(4), ref.RefMesh.grid(31, 17, 1.5)):
        V, F = R.arrays()
        P = port_lib.PortMesh(V, F)
        for v in range(0, R.n, 7):
            a, b = R.fan(v), P.fan(v)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
        for src in ([0], [3, R.n - 2, R.n // 2]):
            for prec in ("single", "double"):
                x = R.ptp(src, precision=prec, labels=True)
                y = P.ptp(src, precision=prec, labels=True)
                assert np.array_equal(bits(x["distances"]), bits(y["distances"]))
                assert np.array_equal(x["labels"], y["labels"])
                assert x["iterations"] == y["iterations"]
