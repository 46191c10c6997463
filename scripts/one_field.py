"""One field on a BASELINE-sized mesh (for ncu captures): grid1001 | height | ico8 | torus."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_08218_b200 as g
which = sys.argv[1] if len(sys.argv) > 1 else "grid1001"
prec = sys.argv[2] if len(sys.argv) > 2 else "single"
if which == "grid1001":
    M, src, lab = g.generate_grid(1001, 1001), [500 * 1001 + 500], False
elif which == "height":
    M = g.heightfield_grid(2048, 2048)
    src = [((2 * b + 1) * 256) * 2048 + (2 * a + 1) * 256 for b in range(4) for a in range(4)]
    lab = True
elif which == "torus":
    M, src, lab = g.generate_torus(1000, 1000), [0], False
else:
    M, src, lab = g.noisy_icosphere(8, 2e-3, 1), [0], False
for _ in range(2):
    r = g.geodesics(M, src, precision=prec, labels=lab)
print(which, prec, "K", r["iterations"], "ms", 1e3 * r["device_seconds"])
