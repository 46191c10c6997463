import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1810_08218_b200 as g
for name in ("ico8", "torus"):
    if name == "torus":
        M = g.generate_torus(1000, 1000)
    else:
        v, f = g.noisy_icosphere_arrays(8, 2e-3, 1)
        M = g.Mesh(v, f)
    n = M.n_vertices
    qs = [[q * (n // 512)] for q in range(32)]
    out = torch.empty((32, n), dtype=torch.float32, device="cuda")
    for groups in (0, 1, 8):
        st = g.batch_geodesics_device(M, qs, out.data_ptr(), groups=groups)
        print(name, "groups", groups, "ms/query", round(1e3 * st[0]["device_seconds"] / 32, 3))
    one = g.geodesics(M, qs[5], precision="single")
    assert np.array_equal(out[5].double().cpu().numpy(), one["distances"]), "batch/auto mismatch"
    print(name, "auto-batch query 5 == single run: ok")
