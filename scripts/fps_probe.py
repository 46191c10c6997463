import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1810_08218_b200 as g
M = g.generate_torus(1000, 1000)
for prec in ("single", "double"):
    g.farthest_point_sampling(M, 4, seed=0, precision=prec)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = g.farthest_point_sampling(M, 200, seed=0, precision=prec)
    print(prec, "fps200 s", round(time.perf_counter() - t, 3), "radius", r["radius"], "samples[:5]", list(r["samples"][:5]), "sum", int(np.sum(r["samples"])))
