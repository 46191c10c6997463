"""GPU parity at the BASELINE configurations' full sizes (SURVEY §8d configs 3-5 and
the 1M-vertex torus field of the bench headline), against the UNMODIFIED reference
(oracle/_ref) run on the same host: bit-exact distances and labels, iteration
counts side by side, and FPS-1000 checked with the survey's cheap argmax test.

Reference: src/ptp.cpp:152-172 (ptp_run), src/sampling.cpp:11-58 (fps, voronoi),
include/geodist/update_kernel.hpp:103-111 (label rule), src/ptp.cpp:64-73 (source
labels).  Each case takes seconds on the GPU and 3-25 s on the host reference."""

import numpy as np
import pytest

from conftest import bits

import paper_1810_08218_b200 as g

pytestmark = pytest.mark.gpu

ref = pytest.importorskip("oracle.ref")
if not ref.available():
    pytest.skip("reference library (oracle/_ref) not built", allow_module_level=True)

HEIGHT_SOURCES = [((2 * b + 1) * 256) * 2048 + (2 * a + 1) * 256 for b in range(4) for a in range(4)]


@pytest.fixture(scope="module")
def torus():
    v, f = g.torus_arrays(1000, 1000)
    return g.Mesh(v, f), ref.RefMesh.torus(1000, 1000)


@pytest.fixture(scope="module")
def height():
    v, f = g.heightfield_arrays(2048, 2048)
    return g.Mesh(v, f), ref.RefMesh.heightfield(2048, 2048)


@pytest.mark.parametrize("prec", ["single", "double"])
def test_torus_1m_field(torus, prec):
    """The bench headline's field: 1000^2 torus, source 0, both precisions; K side by side."""
    M, R = torus
    got = g.geodesics(M, [0], precision=prec)
    want = R.ptp([0], precision=prec)
    assert got["iterations"] == want["iterations"], (got["iterations"], want["iterations"])
    assert got["relax_calls"] == want["relax_calls"]
    assert got["degenerate_calls"] == want["degenerate_calls"]
    assert np.array_equal(bits(got["distances"]), bits(want["distances"]))


@pytest.mark.parametrize("prec", ["single", "double"])
def test_height_field_16_sources_voronoi(height, prec):
    """Config 3: 2048^2 height field, 16 sources with labels (Voronoi), both precisions."""
    M, R = height
    got = g.geodesics(M, HEIGHT_SOURCES, precision=prec, labels=True)
    want = R.ptp(HEIGHT_SOURCES, precision=prec, labels=True)
    assert got["iterations"] == want["iterations"], (got["iterations"], want["iterations"])
    assert got["relax_calls"] == want["relax_calls"]
    assert np.array_equal(bits(got["distances"]), bits(want["distances"]))
    assert np.array_equal(got["labels"], want["labels"])
    assert np.array_equal(g.voronoi(M, HEIGHT_SOURCES, precision=prec), want["labels"])


def test_fps_1000_on_torus(torus):
    """Config 4: FPS with 1000 samples on the 1M torus (fp64, the reference's precision).
    Cheap check: for sampled m, the reference's ptp_run from samples[:m]
    has its argmax (largest distance, lowest index; sampling.cpp:29-36) at samples[m];
    the final labels and covering radius equal the reference's run from all samples."""
    M, R = torus
    r = g.farthest_point_sampling(M, 1000, seed=0)
    s = r["samples"]
    assert s[0] == 0 and len(set(s.tolist())) == 1000
    for m in (1, 10, 100, 500, 999):
        want = R.ptp(s[:m], precision="double", labels=True)
        d = want["distances"]
        assert int(np.argmax(d)) == int(s[m]), (m, int(np.argmax(d)), int(s[m]))
    final = R.ptp(s, precision="double", labels=True)
    assert np.array_equal(r["labels"], final["labels"])
    assert r["radius"] == float(final["distances"].max())


def test_batch_queries_on_torus(torus):
    """Config 5: independent single-source queries s_q = q * floor(n / 512) on the 1M
    torus through the batch scheduler (query 0 alone, the rest as concurrent groups of
    CTAs), a sample of them bit-exact against the reference's single_fp."""
    M, R = torus
    n = M.n_vertices
    queries = [[q * (n // 512)] for q in range(40)]
    out = g.batch_geodesics(M, queries, precision="single")
    for q in (0, 1, 7, 13, 22, 31, 36, 39):
        want = R.ptp(queries[q], precision="single")
        assert out["stats"][q]["iterations"] == want["iterations"], q
        assert out["stats"][q]["relax_calls"] == want["relax_calls"], q
        assert np.array_equal(bits(out["distances"][q]), bits(want["distances"])), q
