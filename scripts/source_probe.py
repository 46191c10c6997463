import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_08218_b200 as g
v, f = g.noisy_icosphere_arrays(8, 2e-3, 1)
M = g.Mesh(v, f)
for s in (0, 1, 11, 12, 5000, 300000, 655361):
    best = None
    for _ in range(2):
        r = g.geodesics(M, [s], precision="single", trace=True)
        if best is None or r["device_seconds"] < best["device_seconds"]:
            best = r
    tr = best["trace"]
    widths = np.array([t["j"] - t["i"] + 1 for t in tr])
    upd = np.array([t["updated"] for t in tr])
    print(f"src {s:7d} K {best['iterations']} U {best['vertex_updates']:9d} ms {1e3*best['device_seconds']:.2f} "
          f"band levels mean {widths.mean():.1f} max {widths.max()} band size mean {upd.mean():.0f} max {upd.max()}")
