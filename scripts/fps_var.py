"""FPS-1000 on the 1000^2 torus, repeated: wall-time spread per precision."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_08218_b200 as g
M = g.generate_torus(1000, 1000)
for prec in ("single", "double", "single"):
    for rep in range(2):
        t = time.perf_counter()
        l0 = g.lib().geodist_kernel_launches()
        r = g.farthest_point_sampling(M, 1000, seed=0, precision=prec)
        print(prec, "wall %.2f s" % (time.perf_counter() - t), "launches", g.lib().geodist_kernel_launches() - l0, flush=True)
