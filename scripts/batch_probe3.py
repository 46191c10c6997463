import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1810_08218_b200 as g
M = g.generate_torus(1000, 1000)
n = M.n_vertices
out = torch.empty((4, n), dtype=torch.float32, device="cuda")
for s in (0, 1953, 3906, 500500):
    for rep in range(2):
        r = g.batch_geodesics_device(M, [[s]], out.data_ptr(), groups=1)
    print("single", s, round(1e3 * r[0]["device_seconds"], 2), r[0]["iterations"], r[0]["vertex_updates"])
st = g.batch_geodesics_device(M, [[0], [0]], out.data_ptr(), groups=1)
print("0,0", 1e3 * st[0]["device_seconds"] / 2)
st = g.batch_geodesics_device(M, [[0], [1953]], out.data_ptr(), groups=1)
print("0,1953", 1e3 * st[0]["device_seconds"] / 2)
r = g.farthest_point_sampling(M, 64, seed=0, precision="single")
import time
t = time.perf_counter()
r = g.farthest_point_sampling(M, 200, seed=0, precision="single")
print("fps 200 rounds s", time.perf_counter() - t, "radius", r["radius"])
