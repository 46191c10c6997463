"""GPU parity: the sm_100a kernels, called through the C ABI, against the
reference's golden vectors (bit-exact distances in both precisions, labels,
K, relax/degenerate counts, band trace, last_change, orderings, FPS), and
against the C restatement on larger synthetic meshes."""

import math

import numpy as np
import pytest

from conftest import FPS_CASES, PTP_CASES, bits, golden

import paper_1810_08218_b200 as g

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["v4", "v4-wide"], autouse=True)
def solver(request, monkeypatch):
    """Run every parity test on both relaxation paths of the solver: the default
    narrow/wide hand-over (v4) and the thread-per-vertex wide-band path forced on
    every iteration (v4-wide)."""
    if request.param.endswith("-wide"):
        monkeypatch.setenv("GEODIST_WIDE", "0")
    else:
        monkeypatch.delenv("GEODIST_WIDE", raising=False)
    return request.param


def mesh_of(gd):
    return g.Mesh(gd["vertices"], gd["faces"])


def test_planar_update_bit_exact():
    gd = golden("planar_update")
    for p, prec in (("s", "single"), ("d", "double")):
        v, s, d = g.planar_update(gd["x1"], gd["x2"], gd["t1"], gd["t2"], precision=prec)
        assert np.array_equal(bits(v), bits(gd[f"value_{p}"]))
        assert np.array_equal(s, gd[f"side_{p}"])
        assert np.array_equal(d, gd[f"degen_{p}"])


@pytest.mark.parametrize("name", PTP_CASES)
@pytest.mark.parametrize("prec", ["single", "double"])
def test_geodesics_bit_exact(name, prec):
    gd = golden(name)
    M = mesh_of(gd)
    p = prec[0]
    labels = f"labels_{p}" in gd
    r = g.geodesics(M, gd["sources"], precision=prec, labels=labels, trace=True)
    assert np.array_equal(bits(r["distances"]), bits(gd[f"dist_{p}"]))
    assert r["iterations"] == int(gd[f"K_{p}"])
    assert r["relax_calls"] == int(gd[f"relax_{p}"])
    assert r["degenerate_calls"] == int(gd[f"degen_{p}"])
    assert r["unreached"] == int(gd["unreached"])
    assert r["rho"] == int(gd["rho"])
    kiju = np.array([[t["k"], t["i"], t["j"], t["updated"]] for t in r["trace"]]).reshape(-1, 4)
    assert np.array_equal(kiju, gd[f"trace_kijU_{p}"])
    assert np.array_equal(bits([t["max_rel_change"] for t in r["trace"]]),
                          bits(gd[f"trace_maxrel_{p}"]))
    assert [t["front_converged"] for t in r["trace"]] == list(gd[f"trace_conv_{p}"])
    assert np.array_equal(r["last_change"], gd[f"last_change_{p}"])
    assert r["vertex_updates"] == int(gd[f"trace_kijU_{p}"][:, 3].sum())
    if labels:
        assert np.array_equal(r["labels"], gd[f"labels_{p}"])
    # without trace the fused fast path must give the same bits
    r2 = g.geodesics(M, gd["sources"], precision=prec, labels=labels)
    assert np.array_equal(bits(r2["distances"]), bits(gd[f"dist_{p}"]))


@pytest.mark.parametrize("name", PTP_CASES)
def test_toplesets_exact(name):
    gd = golden(name)
    t = g.toplesets(mesh_of(gd), gd["sources"])
    assert np.array_equal(t["sorted"], gd["sorted"])
    assert np.array_equal(t["limits"], gd["limits"])
    assert np.array_equal(t["position"], gd["position"])
    assert t["rho"] == int(gd["rho"]) and t["unreached"] == int(gd["unreached"])


@pytest.mark.parametrize("name", PTP_CASES)
def test_reorder_for_bands_exact(name):
    gd = golden(name)
    M = mesh_of(gd)
    P, oon, noo = g.reorder_for_bands(M, gd["sources"])
    assert np.array_equal(oon, gd["old_of_new"])
    assert np.array_equal(noo, gd["new_of_old"])
    assert np.array_equal(P.faces(), gd["reordered_faces"])
    # the caller-ordering entry point (the drop-in's): same permutation, positions
    # permuted on the device
    o = {"sorted": gd["sorted"], "position": gd["position"]}
    P2, oon2, noo2 = g.reorder_for_bands(M, ordering=o)
    assert np.array_equal(oon2, gd["old_of_new"]) and np.array_equal(noo2, gd["new_of_old"])
    assert np.array_equal(P2.faces(), gd["reordered_faces"])
    assert np.array_equal(bits(P2.vertices()), bits(np.asarray(gd["vertices"])[oon2]))
    # test_ptp.cpp:159-180: results bit-identical after un-permutation
    labels = "labels_d" in gd
    src = noo[gd["sources"]]
    r = g.geodesics(P, src, labels=labels)
    assert np.array_equal(bits(r["distances"][noo]), bits(gd["dist_d"]))
    if labels:
        assert np.array_equal(r["labels"][noo], gd["labels_d"])


@pytest.mark.parametrize("name", PTP_CASES)
def test_ptp_with_caller_ordering(name):
    gd = golden(name)
    M = mesh_of(gd)
    o = {"sorted": gd["sorted"], "limits": gd["limits"], "position": gd["position"]}
    labels = "labels_d" in gd
    for p, prec in (("s", "single"), ("d", "double")):
        r = g.geodesics_ordered(M, gd["sources"], o, precision=prec, labels=labels)
        assert np.array_equal(bits(r["distances"]), bits(gd[f"dist_{p}"]))
        assert r["iterations"] == int(gd[f"K_{p}"])


@pytest.mark.parametrize("name", FPS_CASES)
@pytest.mark.parametrize("prec", ["single", "double"])
def test_fps_and_voronoi_exact(name, prec):
    gd = golden(name)
    M = mesh_of(gd)
    p = prec[0]
    r = g.farthest_point_sampling(M, int(gd["m"]), seed=int(gd["seed"]), precision=prec)
    assert np.array_equal(r["samples"], gd[f"samples_{p}"])
    assert np.array_equal(r["labels"], gd[f"labels_{p}"])
    assert r["radius"] == float(gd[f"radius_{p}"])
    assert [h["rho"] for h in r["history"]] == list(gd[f"hist_rho_{p}"])
    assert [h["relax_calls"] for h in r["history"]] == list(gd[f"hist_relax_{p}"])
    assert np.array_equal(bits([h["radius"] for h in r["history"]]), bits(gd[f"hist_radius_{p}"]))
    assert [h["picked"] for h in r["history"]] == list(gd[f"hist_picked_{p}"])
    lab = g.voronoi(M, gd[f"samples_{p}"], precision=prec)
    assert np.array_equal(lab, gd[f"voronoi_{p}"])


def polar_arrays(spokes, rings, twist=0.37):
    """Wheel mesh: a centre of valence `spokes` (> 7 exercises the CSR overflow path)."""
    v = [[0.0, 0.0, 0.0]]
    for r in range(1, rings + 1):
        for s in range(spokes):
            a = 2 * np.pi * s / spokes + twist * r
            v.append([r * np.cos(a), r * np.sin(a), 0.05 * r * np.sin(3 * a)])
    f = []
    ring = lambda r, s: 1 + (r - 1) * spokes + (s % spokes)
    for s in range(spokes):
        f.append([0, ring(1, s), ring(1, s + 1)])
    for r in range(1, rings):
        for s in range(spokes):
            a, b, c, d = ring(r, s), ring(r, s + 1), ring(r + 1, s + 1), ring(r + 1, s)
            f.append([a, d, c])
            f.append([a, c, b])
    return np.array(v), np.array(f, np.int32)


SYNTH = [
    ("wheel12", lambda: polar_arrays(12, 9), [[0], [5, 40]]),
    ("wheel23", lambda: polar_arrays(23, 6), [[0], [3]]),
    # 5000 claims by one CTA in one iteration: the on-chip claim list spills to global
    ("wheel5000", lambda: polar_arrays(5000, 3), [[0], [7, 12000]]),
    # 9000 claims by one CTA in one iteration: beyond the CTA's global list as first
    # sized, so the field is abandoned (err 2) and redone with full-size lists; from
    # the centre (iteration-0 claims) and from a spoke (the centre claims at k = 1)
    ("wheel9000", lambda: polar_arrays(9000, 3), [[0], [7], [7, 20000]]),
    # a first topleset wider than the narrow path's record cache on every CTA (20000 > 148 x
    # 127): the BFS pre-pass caches rows into wrapping slots, the field goes wide at once
    ("wheel20000", lambda: polar_arrays(20000, 2), [[0]]),
    ("ico5", lambda: g.icosphere_arrays(5), [[0], [5, 700, 9000]]),
    ("noisy_ico6", lambda: g.noisy_icosphere_arrays(6, 2e-3, 1), [[0], [1, 20000, 33333, 40000]]),
    ("torus64x48", lambda: g.torus_arrays(64, 48), [[0], [17, 1500, 3000]]),
    ("height96", lambda: g.heightfield_arrays(96, 96, 20.0, 9.7, 13.1), [[0], [100, 5000, 9000]]),
    ("grid40_shear2", lambda: g.grid_arrays(40, 40, 2.0), [[820], [0, 1599]]),
    # more toplesets than the on-chip limits ring holds (rho ~ 2600 > 1024 levels)
    ("strip2600x3", lambda: g.grid_arrays(2600, 3, 0.0), [[0], [1300, 7799]]),
]


@pytest.mark.parametrize("name,make,sources", SYNTH, ids=[s[0] for s in SYNTH])
def test_synthetic_vs_restatement(port_lib, name, make, sources):
    v, f = make()
    M = g.Mesh(v, f)
    P = port_lib.PortMesh(v, f)
    for src in sources:
        for prec in ("single", "double"):
            want = P.ptp(src, precision=prec, labels=True)
            got = g.geodesics(M, src, precision=prec, labels=True)
            assert np.array_equal(bits(got["distances"]), bits(want["distances"])), (src, prec)
            assert np.array_equal(got["labels"], want["labels"])
            assert got["iterations"] == want["iterations"]
            assert got["relax_calls"] == want["relax_calls"]
            assert got["degenerate_calls"] == want["degenerate_calls"]


def test_claim_overflow_batch_and_fps_redo(port_lib):
    """The claim-list overflow redo on the batch and FPS entry points: a
    9000-spoke wheel, fields equal the single-field path / the restatement."""
    v, f = polar_arrays(9000, 3)
    M = g.Mesh(v, f)
    queries = [[0], [7], [9001, 18000]]
    out = g.batch_geodesics(M, queries, precision="single", labels=True, groups=2)
    for q, src in enumerate(queries):
        one = g.geodesics(M, src, precision="single", labels=True)
        assert np.array_equal(bits(out["distances"][q]), bits(one["distances"]))
        assert np.array_equal(out["labels"][q], one["labels"])
    r = g.farthest_point_sampling(M, 4, seed=7)
    want = port_lib.PortMesh(v, f).fps(4, seed=7)
    assert list(r["samples"]) == list(want["samples"])
    assert np.array_equal(r["labels"], want["labels"])


def test_batch_equals_single_runs():
    v, f = g.noisy_icosphere_arrays(5, 2e-3, 1)
    M = g.Mesh(v, f)
    queries = [[q * 97] for q in range(9)] + [[3, 5000, 9000]]
    for prec in ("single", "double"):
        for groups in (1, 3, 4):
            out = g.batch_geodesics(M, queries, precision=prec, labels=True, groups=groups)
            for q, src in enumerate(queries):
                one = g.geodesics(M, src, precision=prec, labels=True)
                assert np.array_equal(bits(out["distances"][q]), bits(one["distances"]))
                assert np.array_equal(out["labels"][q], one["labels"])
                assert out["stats"][q]["iterations"] == one["iterations"]
                assert out["stats"][q]["relax_calls"] == one["relax_calls"]


def test_batch_wide_bands_equal_single_runs():
    """Batched fields whose bands exceed the record cache (600^2 torus): one group (the
    per-query narrow/wide launch sequence), several groups (the combined kernel on 37-74
    CTAs per field) and the automatic choice all equal the single-field path."""
    v, f = g.torus_arrays(600, 600)
    M = g.Mesh(v, f)
    n = len(v)
    queries = [[0], [n // 3], [2 * n // 3 + 17]]
    single = [g.geodesics(M, q, precision="single") for q in queries]
    for groups in (0, 1, 2, 4):
        out = g.batch_geodesics(M, queries, precision="single", groups=groups)
        for q in range(len(queries)):
            assert np.array_equal(bits(out["distances"][q]), bits(single[q]["distances"])), groups
            assert out["stats"][q]["iterations"] == single[q]["iterations"]


def test_observer_monotone():
    # test_ptp.cpp:60-74: distances never increase across iterations
    M = g.generate_grid(9, 9, 2.0)
    prev = np.full(81, np.inf)
    ks = []

    def obs(k, d):
        nonlocal prev
        assert np.all(d <= prev)
        prev = d
        ks.append(k)

    r = g.geodesics(M, [40], observer=obs)
    assert ks == list(range(1, r["iterations"] + 1))
    assert np.array_equal(prev, r["distances"])


def test_errors_match_reference():
    M = g.generate_grid(5, 5)
    with pytest.raises(ValueError, match="empty source set"):
        g.geodesics(M, [])
    with pytest.raises(ValueError, match="out of range"):
        g.geodesics(M, [25])
    with pytest.raises(ValueError, match="duplicate source"):
        g.geodesics(M, [3, 3])
    with pytest.raises(ValueError, match="epsilon must be positive"):
        g.geodesics(M, [0], epsilon=0.0)
    with pytest.raises(ValueError, match="precision"):
        g.geodesics(M, [0], precision="half")
    with pytest.raises(ValueError, match="sample count"):
        g.farthest_point_sampling(M, 0)
    with pytest.raises(ValueError, match="seed"):
        g.farthest_point_sampling(M, 2, seed=99)
    with pytest.raises(ValueError, match="empty sample"):
        g.voronoi(M, [])
    o = g.toplesets(M, [0])
    with pytest.raises(ValueError, match="does not match the source set"):
        g.geodesics_ordered(M, [1], o)


def test_reference_properties():
    # test_ptp.cpp:44-58 sandwich, :182-199 labels, :243-265 K/rho regime
    for shear in (0.0, 2.0):
        M = g.generate_grid(9, 7, shear)
        r = g.geodesics(M, [0])
        exact = g.grid_reference(M, [0])
        assert np.all(r["distances"] >= exact * (1 - 1e-12))
    M = g.generate_grid(9, 5)
    r = g.geodesics(M, [0, 8], labels=True)
    assert r["labels"][0] == 0 and r["labels"][8] == 1
    for j in range(5):
        assert r["labels"][j * 9 + 1] == 0 and r["labels"][j * 9 + 7] == 1
    M = g.generate_grid(41, 41)
    c = 20 * 41 + 20
    rep = g.mape(g.geodesics(M, [c])["distances"], g.grid_reference(M, [c]), [c])
    assert rep["mape"] < 3.5
    S = g.generate_icosphere(3)
    rep = g.mape(g.geodesics(S, [0])["distances"], g.sphere_reference(S, [0]), [0])
    assert rep["mape"] < 3.0


def test_fast_path_arithmetic_is_ieee():
    """The straight-line div.rn / sqrt.rn sequences the kernels use (fp32 and fp64,
    ptp_common.cuh) return the IEEE correctly rounded result on every operand they
    accept: 2^26 pseudo-random pairs over a wide exponent range."""
    from paper_1810_08218_b200 import _capi
    counts = np.zeros(8, np.int64)
    g.check(_capi.lib().geodist_selftest_arith(1 << 26, 12345, counts))
    acc, bad = counts[0::2], counts[1::2]
    assert (acc > (1 << 24)).all(), counts
    assert (bad == 0).all(), counts


def test_degenerate_source_sets(port_lib):
    """Every vertex a source (one topleset, no iteration), and a source on an isolated
    vertex next to a component it cannot reach."""
    v, f = g.icosphere_arrays(2)
    M = g.Mesh(v, f)
    P = port_lib.PortMesh(v, f)
    allv = list(range(len(v)))
    for prec in ("single", "double"):
        got = g.geodesics(M, allv, precision=prec, labels=True)
        want = P.ptp(allv, precision=prec, labels=True)
        assert np.array_equal(bits(got["distances"]), bits(want["distances"]))
        assert np.array_equal(got["labels"], want["labels"])
        assert got["iterations"] == want["iterations"]
    v2 = np.vstack([v, [[3.0, 3.0, 3.0]]])
    M2 = g.Mesh(v2, f)
    P2 = port_lib.PortMesh(v2, f)
    for src in ([len(v)], [0, len(v)]):
        for prec in ("single", "double"):
            got = g.geodesics(M2, src, precision=prec, labels=True)
            want = P2.ptp(src, precision=prec, labels=True)
            assert np.array_equal(bits(got["distances"]), bits(want["distances"]))
            assert np.array_equal(got["labels"], want["labels"])
            assert got["unreached"] == want["unreached"]


def test_narrow_wide_handover_parity():
    """A field whose band grows past the record cache and shrinks back (600^2 torus: the
    band exceeds 511 x 148 positions in iterations 239-613 of 706, so the narrow-only
    launch hands over to the wide-only launch and back), against the unmodified
    reference, both precisions; K and relax counts too."""
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library not built")
    v, f = g.torus_arrays(600, 600)
    M = g.Mesh(v, f)
    R = ref.RefMesh.from_arrays(v, f)
    for prec in ("single", "double"):
        got = g.geodesics(M, [0], precision=prec)
        want = R.ptp([0], precision=prec, workers=0)
        assert np.array_equal(bits(got["distances"]), bits(want["distances"])), prec
        assert got["iterations"] == want["iterations"]
        assert got["relax_calls"] == want["relax_calls"]


def test_fps_across_handover_parity():
    """FPS rounds (the fixed per-round launch sequence) on the 600^2 torus: the first
    rounds' samples, labels and covering radius equal the reference's (fp64)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library not built")
    v, f = g.torus_arrays(600, 600)
    M = g.Mesh(v, f)
    R = ref.RefMesh.from_arrays(v, f)
    got = g.farthest_point_sampling(M, 3, seed=0)
    want = R.fps(3, seed=0, precision="double", workers=0)
    assert list(got["samples"]) == list(want["samples"])
    assert np.array_equal(got["labels"], want["labels"])
    assert got["radius"] == want["radius"]


def test_malformed_orderings_rejected():
    """ptp_run / reorder_for_bands with an ordering that is not one of this
    mesh's (decreasing limits, a position array inconsistent with sorted) fail with the
    reference's invalid_argument text instead of reaching device memory."""
    v, f = g.icosphere_arrays(2)
    M = g.Mesh(v, f)
    t = g.toplesets(M, [0])
    bad = {"sorted": t["sorted"], "limits": t["limits"].copy(), "position": t["position"]}
    bad["limits"][2], bad["limits"][3] = bad["limits"][3], bad["limits"][2]
    with pytest.raises(ValueError, match="ordering"):
        g.geodesics_ordered(M, [0], bad)
    pos = t["position"].copy()
    pos[t["sorted"][3]] = 7
    with pytest.raises(ValueError, match="ordering"):
        g.reorder_for_bands(M, ordering={"sorted": t["sorted"], "position": pos})
