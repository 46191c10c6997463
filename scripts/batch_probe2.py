import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1810_08218_b200 as g
v, f = g.noisy_icosphere_arrays(8, 2e-3, 1)
M = g.Mesh(v, f)
n = M.n_vertices
out = torch.empty((8, n), dtype=torch.float32, device="cuda")
for nq in (1, 2, 4, 8):
    for rep in range(2):
        st = g.batch_geodesics_device(M, [[0]] * nq, out.data_ptr(), groups=1)
    print("same source x", nq, "ms/query", 1e3 * st[0]["device_seconds"] / nq, [s["iterations"] for s in st])
st = g.batch_geodesics_device(M, [[0], [5000], [0]], out.data_ptr(), groups=1)
print("0,5000,0", 1e3 * st[0]["device_seconds"] / 3, [s["iterations"] for s in st])
for s in (0, 5000, 300000):
    r = g.batch_geodesics_device(M, [[s]], out.data_ptr(), groups=1)
    print("single", s, 1e3 * r[0]["device_seconds"], r[0]["iterations"])
