import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1810_08218_b200 as g
M = g.generate_torus(1000, 1000)
n = M.n_vertices
qs = [[q * (n // 512)] for q in range(32)]
out = torch.empty((32, n), dtype=torch.float32, device="cuda")
for nq in (1, 2, 4, 8, 16, 32):
    st = g.batch_geodesics_device(M, qs[:nq], out.data_ptr(), groups=1)
    print("nq", nq, "ms/query", round(1e3 * st[0]["device_seconds"] / nq, 3), "K", [s["iterations"] for s in st][-3:])
for q in (8, 16, 24, 31):
    st = g.batch_geodesics_device(M, [qs[q]], out.data_ptr(), groups=1)
    print("single q", q, round(1e3 * st[0]["device_seconds"], 3), st[0]["iterations"], st[0]["vertex_updates"])
