"""Mesh creation time, device fan build vs host build (GEODIST_HOST_BUILD=1), on the
BASELINE meshes; wall clock of Mesh(v, f) (validation, fan build, uploads)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_08218_b200 as g

out = {}
g.Mesh(*g.icosphere_arrays(2))  # context + library warm-up
for name, make in [("noisy_icosphere8", lambda: g.noisy_icosphere_arrays(8, 2e-3, 1)),
                   ("torus1000", lambda: g.torus_arrays(1000, 1000)),
                   ("height2048", lambda: g.heightfield_arrays(2048, 2048))]:
    v, f = make()
    row = {}
    for mode in ("0", "1"):
        os.environ["GEODIST_HOST_BUILD"] = mode
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            M = g.Mesh(v, f)
            best = min(best, time.perf_counter() - t)
            del M
        row["host_build_s" if mode == "1" else "device_build_s"] = best
    os.environ["GEODIST_HOST_BUILD"] = "0"
    c, r, d = g.Mesh(v, f).fans()
    hc, hr, hd = g.build_fans(v, f)
    row["equal_to_host"] = bool(np.array_equal(c, hc) and np.array_equal(r, hr) and np.array_equal(d, hd))
    out[name] = row
    print(name, row, flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/mesh_build.json", "w"), indent=1)
