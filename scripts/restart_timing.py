"""Where the narrow iteration's restart goes: per iteration, thread 0's barrier release
(slot 2) -> end of post/publish (slot 8) -> the next iteration's start (slot 0), from the
GEODIST_DEBUG_TIMING buffer of one icosphere-8 field (narrow iterations only)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GEODIST_DEBUG_TIMING"] = "2000"
import paper_1810_08218_b200 as g  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "single"
v, f = g.noisy_icosphere_arrays(8, 2e-3, 1)
M = g.Mesh(v, f)
os.makedirs("gpurun_out", exist_ok=True)
for _ in range(2):
    r = g.geodesics(M, [0], precision=prec)
print("K", r["iterations"], "ms", 1e3 * r["device_seconds"])
raw = open("gpurun_out/dbg_timing.bin", "rb").read()
it, nb = np.frombuffer(raw[:8], np.int32)
t = np.frombuffer(raw[8:], np.uint64).reshape(it, nb, -1).astype(np.int64)
ok = (t[:, :, 0] > 0).all(axis=1) & (t[:, :, 18] == 0).all(axis=1)
idx = np.nonzero(ok)[0]
idx = idx[idx + 1 < it]
idx = idx[ok[idx + 1]]
rel, pub, nxt = t[idx, :, 2], t[idx, :, 8], t[idx + 1, :, 0]
good = (pub >= rel) & (pub - rel < 100000)
print("narrow iterations", len(idx))
print("release -> publish end ns: mean %.0f" % (pub - rel)[good].mean())
print("publish end -> next start ns: mean %.0f" % (nxt - pub)[good].mean())
print("release -> next start ns: mean %.0f" % (nxt - rel).mean())
