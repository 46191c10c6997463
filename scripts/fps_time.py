"""BASELINE configs[3]: farthest-point sampling of 1000 samples on the 1000^2 torus, both
precisions (wall clock of the whole call: all rounds run back to back on the device).

  python scripts/fps_time.py [count]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_08218_b200 as g  # noqa: E402

cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
M = g.generate_torus(1000, 1000)
out = {"count": cnt, "mesh": "torus 1000x1000 (1,000,000 vertices)", "seed": 0}
for prec in ("double", "single"):
    g.farthest_point_sampling(M, 4, seed=0, precision=prec)  # warm-up
    t = time.perf_counter()
    r = g.farthest_point_sampling(M, cnt, seed=0, precision=prec)
    dt = time.perf_counter() - t
    out[prec] = {"seconds": dt, "ms_per_round": 1e3 * dt / cnt, "radius": float(r["radius"]),
                 "last_samples": [int(x) for x in r["samples"][-3:]]}
print(json.dumps(out, indent=1))
