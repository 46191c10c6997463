"""FPS on the 1000^2 torus: per-round iterations / relax calls, and wall time split."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_08218_b200 as g
prec = sys.argv[1] if len(sys.argv) > 1 else "double"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
M = g.generate_torus(1000, 1000)
g.farthest_point_sampling(M, 2, seed=0, precision=prec)
t = time.perf_counter()
r = g.farthest_point_sampling(M, count, seed=0, precision=prec)
wall = time.perf_counter() - t
h = r["history"]
K = np.array([x["iterations"] for x in h]); C = np.array([x["relax_calls"] for x in h]); rho = np.array([x["rho"] for x in h])
for lo, hi in ((0, 10), (10, 100), (100, 500), (500, count)):
    if lo < count:
        s = slice(lo, min(hi, count))
        print(f"rounds {lo}-{hi}: K mean {K[s].mean():.0f} rho mean {rho[s].mean():.0f} relax/round {C[s].mean()/1e6:.1f} M")
print(f"total wall {wall:.2f} s, {1e3*wall/count:.2f} ms/round, total relax {C.sum()/1e9:.2f} G, total K {K.sum()}")
