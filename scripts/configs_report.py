"""BASELINE.json configurations on one B200, with the unmodified reference (oracle/_ref,
OpenMP over all host threads) timed beside them on the same box.

  python scripts/configs_report.py [out.json]

1. icosphere subdiv-3 single source: GPU and CPU, bit-exactness, K
2. noisy icosphere subdiv-8 (sigma 2e-3) single source: GPU fp32/fp64 and CPU
3. 2048^2 height field, 16 sources + Voronoi labels: GPU fp32/fp64, CPU fp64 (one run),
   label mismatches GPU fp32 vs CPU fp64 and GPU fp64 vs CPU fp64
4. FPS 1000 samples on the 1000^2 torus: GPU total (fp64, the reference's precision,
   and fp32); CPU: the first rounds (extrapolated by the measured per-round time) and
   the GPU sample list checked against the CPU's for those rounds
5. 512 independent single-source queries on the torus: GPU per-query time (all 512 on
   one GPU, groups chosen by the library) and CPU per query (2 queries)
Times are device time (CUDA events) for the GPU unless marked wall; CPU times are the
reference's own timers (compute_toplesets + ptp_run) or wall clock for fps.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1810_08218_b200 as g  # noqa: E402
from oracle import ref  # noqa: E402

out = {"threads": ref.max_threads() if ref.available() else None}


def gpu_field(M, src, prec, labels=False, reps=2):
    best = None
    for _ in range(reps):
        r = g.geodesics(M, src, precision=prec, labels=labels)
        if best is None or r["device_seconds"] < best["device_seconds"]:
            best = r
    return best


def cpu_field(R, src, prec, labels=False):
    r = R.ptp(src, precision=prec, labels=labels, workers=0)
    return r, 1e3 * (r["wall_seconds"] + r["toplesets_seconds"])


def bits_equal(a, b):
    return bool(np.array_equal(np.asarray(a, np.float64).view(np.int64),
                               np.asarray(b, np.float64).view(np.int64)))


# 1 -------------------------------------------------------------------------------
v, f = g.icosphere_arrays(3)
M = g.Mesh(v, f)
R = ref.RefMesh.from_arrays(v, f)
c1 = {}
for prec in ("double", "single"):
    gr = gpu_field(M, [0], prec)
    cr, cms = cpu_field(R, [0], prec)
    c1[prec] = {"gpu_ms": 1e3 * gr["device_seconds"], "cpu_ms": cms, "K_gpu": gr["iterations"],
                "K_cpu": cr["iterations"], "bit_exact": bits_equal(gr["distances"], cr["distances"])}
diag = float(np.linalg.norm(v.max(0) - v.min(0)))
c1["fp32_vs_fp64_max_abs_err_over_diag"] = float(
    np.max(np.abs(gpu_field(M, [0], "single")["distances"] - R.ptp([0], precision="double")["distances"])) / diag)
out["1_icosphere3"] = c1

# 2 -------------------------------------------------------------------------------
v, f = g.noisy_icosphere_arrays(8, 2e-3, 1)
M = g.Mesh(v, f)
R = ref.RefMesh.from_arrays(v, f)
c2 = {}
for prec in ("single", "double"):
    gr = gpu_field(M, [0], prec, reps=3)
    cr, cms = cpu_field(R, [0], prec)
    c2[prec] = {"gpu_ms": 1e3 * gr["device_seconds"], "cpu_ms": cms, "K_gpu": gr["iterations"],
                "K_cpu": cr["iterations"], "bit_exact": bits_equal(gr["distances"], cr["distances"]),
                "U": gr["vertex_updates"], "C": gr["relax_calls"]}
diag = float(np.linalg.norm(v.max(0) - v.min(0)))
g32 = gpu_field(M, [0], "single", reps=1)["distances"]
g64 = gpu_field(M, [0], "double", reps=1)["distances"]  # bit-exact with the reference's fp64
fin = np.isfinite(g64)
c2["fp32_vs_fp64_max_abs_err_over_diag"] = float(np.max(np.abs(g32[fin] - g64[fin])) / diag)
out["2_noisy_icosphere8"] = c2
del M, R

# 3 -------------------------------------------------------------------------------
v, f = g.heightfield_arrays(2048, 2048)
M = g.Mesh(v, f)
R = ref.RefMesh.from_arrays(v, f)
src = [((2 * b + 1) * 256) * 2048 + (2 * a + 1) * 256 for b in range(4) for a in range(4)]
c3 = {}
cr64, cms64 = cpu_field(R, src, "double", labels=True)
diag = float(np.linalg.norm(v.max(0) - v.min(0)))
for prec in ("single", "double"):
    gr = gpu_field(M, src, prec, labels=True, reps=1)
    c3[prec] = {"gpu_ms": 1e3 * gr["device_seconds"], "K_gpu": gr["iterations"],
                "label_mismatches_vs_cpu_fp64": int((gr["labels"] != cr64["labels"]).sum()),
                "max_abs_err_over_diag_vs_cpu_fp64": float(
                    np.max(np.abs(gr["distances"] - cr64["distances"])) / diag)}
c3["cpu_fp64_ms"] = cms64
c3["K_cpu_fp64"] = cr64["iterations"]
c3["fp64_bit_exact"] = bits_equal(gpu_field(M, src, "double", labels=True, reps=1)["distances"],
                                  cr64["distances"])
out["3_heightfield2048_16src_voronoi"] = c3
del M, R

# 4 -------------------------------------------------------------------------------
v, f = g.torus_arrays(1000, 1000)
M = g.Mesh(v, f)
R = ref.RefMesh.from_arrays(v, f)
c4 = {}
diag = float(np.linalg.norm(v.max(0) - v.min(0)))
g32 = gpu_field(M, [0], "single", reps=1)["distances"]
g64 = gpu_field(M, [0], "double", reps=1)["distances"]
c4["single_field_fp32_vs_fp64_max_abs_err_over_diag"] = float(np.max(np.abs(g32 - g64)) / diag)
for prec in ("double", "single"):
    g.farthest_point_sampling(M, 4, seed=0, precision=prec)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = g.farthest_point_sampling(M, 1000, seed=0, precision=prec)
    c4[f"gpu_{prec}_s_wall"] = time.perf_counter() - t
    c4[f"gpu_{prec}_radius"] = r["radius"]
    if prec == "double":
        gpu_samples = np.asarray(r["samples"])
prefix = 3
t = time.perf_counter()
cf = R.fps(prefix, seed=0, precision="double", workers=0)
cpu_s = time.perf_counter() - t
c4["cpu_prefix_rounds"] = prefix
c4["cpu_prefix_s_wall"] = cpu_s
c4["cpu_extrapolated_1000_s"] = cpu_s / prefix * 1000
c4["prefix_samples_match_fp64"] = bool(np.array_equal(cf["samples"], gpu_samples[:prefix]))
out["4_fps1000_torus"] = c4

# 5 -------------------------------------------------------------------------------
n = M.n_vertices
qs = [[q * (n // 512)] for q in range(512)]
buf = torch.empty((64, n), dtype=torch.float32, device="cuda")
g.batch_geodesics_device(M, qs[:2], buf.data_ptr())  # warm
torch.cuda.synchronize()
dev = 0.0
t = time.perf_counter()
for b in range(0, 512, 64):
    st = g.batch_geodesics_device(M, qs[b:b + 64], buf.data_ptr())
    dev += st[0]["device_seconds"]
torch.cuda.synchronize()
wall = time.perf_counter() - t
cpu = [cpu_field(R, qs[q], "single")[1] for q in (0, 1)]
out["5_512_queries_torus"] = {"gpu_ms_per_query": 1e3 * dev / 512, "gpu_wall_s": wall,
                              "cpu_ms_per_query": float(np.mean(cpu)),
                              "cpu_extrapolated_512_s": float(np.mean(cpu)) * 512 / 1e3,
                              "note": "one GPU; the bench's --gpus N run shards fields over N ranks"}

path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "configs.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
