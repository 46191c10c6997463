"""Batched independent queries on one GPU: device time per query vs groups (config 5 shape)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1810_08218_b200 as g

mesh_name = sys.argv[1] if len(sys.argv) > 1 else "torus"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 16
labels = False
if mesh_name == "torus":
    M = g.generate_torus(1000, 1000)
elif mesh_name == "height":
    M = g.heightfield_grid(2048, 2048)
else:
    v, f = g.noisy_icosphere_arrays(8, 2e-3, 1)
    M = g.Mesh(v, f)
n = M.n_vertices
qs = [[q * (n // 512)] for q in range(nq)]
out = torch.empty((nq, n), dtype=torch.float32, device="cuda")
res = {}
for groups in (1, 2, 4, 8, 16, 0):
    g.batch_geodesics_device(M, qs[:max(groups, 3)], out.data_ptr(), groups=groups)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    st = g.batch_geodesics_device(M, qs, out.data_ptr(), groups=groups)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    res[groups] = {"device_ms_per_query": 1e3 * st[0]["device_seconds"] / nq,
                   "wall_ms_per_query": 1e3 * wall / nq, "K": [s["iterations"] for s in st][:4]}
singles = [1e3 * g.batch_geodesics_device(M, [q], out.data_ptr(), groups=1)[0]["device_seconds"]
           for q in qs]
res["single_mean_ms"] = sum(singles) / len(singles)
res["single_ms"] = singles[:8]
print(json.dumps({"mesh": mesh_name, "nq": nq, "res": res}, indent=1))
