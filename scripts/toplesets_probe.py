"""compute_toplesets on the device (exact reference order) and the drop-in's two-call
path (compute_toplesets -> ptp_run with that ordering), timed on the BASELINE meshes
next to the reference's own compute_toplesets (oracle/_ref, host).

    python scripts/toplesets_probe.py > profiles/round2/toplesets.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_08218_b200 as g  # noqa: E402
from oracle import ref  # noqa: E402

HEIGHT_SRC = [((2 * b + 1) * 256) * 2048 + (2 * a + 1) * 256 for b in range(4) for a in range(4)]
cases = [("torus1000_src0", lambda: g.torus_arrays(1000, 1000), lambda: ref.RefMesh.torus(1000, 1000), [0]),
         ("height2048_16src", lambda: g.heightfield_arrays(2048, 2048),
          lambda: ref.RefMesh.heightfield(2048, 2048), HEIGHT_SRC)]
out = {}
for name, mk, mkref, src in cases:
    v, f = mk()
    M = g.Mesh(v, f)
    g.toplesets(M, src)  # warm (scratch allocation)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        o = g.toplesets(M, src)
        ts.append(time.perf_counter() - t)
    R = mkref()
    want = R.toplesets(src)
    exact = (np.array_equal(o["sorted"], want["sorted"]) and
             np.array_equal(o["limits"], want["limits"]) and
             np.array_equal(o["position"], want["position"]))
    # the drop-in's two-call path: ordering from the device, then ptp_run with it
    two = []
    for _ in range(3):
        t = time.perf_counter()
        o2 = g.toplesets(M, src)
        r = g.geodesics_ordered(M, src, o2, precision="single", labels=len(src) > 1)
        two.append(time.perf_counter() - t)
    fused = g.geodesics(M, src, precision="single", labels=len(src) > 1)
    out[name] = {"n": len(v), "rho": o["rho"], "gpu_toplesets_ms": 1e3 * min(ts),
                 "ref_toplesets_ms": 1e3 * want["seconds"], "exact_order": bool(exact),
                 "two_call_ms_wall": 1e3 * min(two),
                 "fused_field_device_ms": 1e3 * fused["device_seconds"],
                 "two_call_equals_fused": bool(np.array_equal(r["distances"], fused["distances"]))}
    print(name, out[name], file=sys.stderr)
print(json.dumps(out, indent=1))
