"""One torus-1000 single-source field (wide bands), for profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_08218_b200 as g
prec = sys.argv[1] if len(sys.argv) > 1 else "single"
M = g.generate_torus(1000, 1000)
for _ in range(2):
    r = g.geodesics(M, [0], precision=prec)
print("K", r["iterations"], "ms", 1e3 * r["device_seconds"])
