"""Torus: per-source single-field device time vs the same sources in one batch call."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1810_08218_b200 as g

M = g.generate_torus(1000, 1000)
n = M.n_vertices
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
qs = [[q * (n // 512)] for q in range(nq)]
out = torch.empty((nq, n), dtype=torch.float32, device="cuda")
g.geodesics(M, qs[0], precision="single")
single = []
for q in qs:
    r = g.geodesics(M, q, precision="single")
    single.append((q[0], r["iterations"], round(1e3 * r["device_seconds"], 2)))
res = {"single": single}
for groups in (1, 2):
    l0 = g.kernel_launches() if hasattr(g, "kernel_launches") else None
    st = g.batch_geodesics_device(M, qs, out.data_ptr(), groups=groups)
    torch.cuda.synchronize()
    res[f"batch_g{groups}_ms_per_query"] = 1e3 * st[0]["device_seconds"] / nq
    res[f"batch_g{groups}_K"] = [s["iterations"] for s in st]
print(json.dumps(res))
