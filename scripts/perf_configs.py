"""Time the SURVEY §8d configurations on one GPU (device time per field, K, U, C)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_08218_b200 as g  # noqa: E402

which = sys.argv[1:] or ["grid1001", "ico8", "torus", "height", "fps", "batch"]
out = {}


def field(M, src, prec, labels=False, reps=3):
    best = None
    for _ in range(reps):
        r = g.geodesics(M, src, precision=prec, labels=labels)
        best = r if best is None or r["device_seconds"] < best["device_seconds"] else best
    return {"ms": 1e3 * best["device_seconds"], "K": best["iterations"], "rho": best["rho"],
            "U": best["vertex_updates"], "C": best["relax_calls"]}


if "grid1001" in which:
    M = g.generate_grid(1001, 1001)
    c = 500 * 1001 + 500
    out["grid1001_center"] = {p: field(M, [c], p) for p in ("single", "double")}
if "ico8" in which:
    M = g.noisy_icosphere(8, 2e-3, 1)
    out["ico8_noisy"] = {p: field(M, [0], p) for p in ("single", "double")}
if "torus" in which:
    M = g.generate_torus(1000, 1000)
    out["torus1000"] = {p: field(M, [0], p, reps=2) for p in ("single", "double")}
if "height" in which or "height64" in which:
    M = g.heightfield_grid(2048, 2048)
    src = [((2 * b + 1) * 256) * 2048 + (2 * a + 1) * 256 for b in range(4) for a in range(4)]
    precs = ("single",) if "height64" not in which else ("single", "double")
    out["height2048_16src_labels"] = {p: field(M, src, p, labels=True, reps=1) for p in precs}
if "fps" in which:
    M = g.generate_torus(1000, 1000)
    t = time.perf_counter()
    r = g.farthest_point_sampling(M, 16, seed=0, precision="single")
    out["torus_fps16_single_s"] = time.perf_counter() - t
if "fps32" in which:
    # ab.sh-friendly: {precision: {"ms": wall ms for 32 FPS rounds}}
    M = g.generate_torus(1000, 1000)
    out["torus_fps32"] = {}
    for prec in ("single", "double"):
        g.farthest_point_sampling(M, 2, seed=0, precision=prec)
        t = time.perf_counter()
        g.farthest_point_sampling(M, 32, seed=0, precision=prec)
        out["torus_fps32"][prec] = {"ms": 1e3 * (time.perf_counter() - t)}
if "batch" in which:
    M = g.generate_torus(1000, 1000)
    n = M.n_vertices
    qs = [[q * (n // 512)] for q in range(32)]
    for groups in (1, 2, 4):
        res = g.batch_geodesics(M, qs, precision="single", groups=groups)
        t = time.perf_counter()
        res = g.batch_geodesics(M, qs, precision="single", groups=groups)
        out[f"torus_batch32_groups{groups}_ms_per_query"] = 1e3 * (time.perf_counter() - t) / len(qs)
print(json.dumps(out, indent=1))
