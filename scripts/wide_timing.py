"""Per-iteration anatomy of the wide-band iterations of one field (GEODIST_DEBUG_TIMING):
newest-topleset loop, older-band work, barrier; max over CTAs.

  python scripts/wide_timing.py [single|double] [torus|height]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GEODIST_DEBUG_TIMING"] = "3000"
import paper_1810_08218_b200 as g  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "single"
which = sys.argv[2] if len(sys.argv) > 2 else "torus"
if which == "torus":
    M, src, lab = g.generate_torus(1000, 1000), [0], False
else:
    M = g.heightfield_grid(2048, 2048)
    src = [((2 * b + 1) * 256) * 2048 + (2 * a + 1) * 256 for b in range(4) for a in range(4)]
    lab = True
os.makedirs("gpurun_out", exist_ok=True)
for _ in range(2):
    r = g.geodesics(M, src, precision=prec, labels=lab)
print(which, prec, "K", r["iterations"], "device ms", 1e3 * r["device_seconds"])
raw = open("gpurun_out/dbg_timing.bin", "rb").read()
it, nb = np.frombuffer(raw[:8], np.int32)
t = np.frombuffer(raw[8:], np.uint64).reshape(it, nb, -1).astype(np.int64)
valid = (t[:, :, 0] > 0).all(axis=1)
idx = np.nonzero(valid)[0]
t = t[valid]
wide = (t[:, :, 18] == 1).all(axis=1)
print("iterations recorded", len(t), "wide", int(wide.sum()))
for name, sel in (("wide", wide), ("narrow", ~wide)):
    if not sel.any():
        continue
    x = t[sel]
    base = x[:, :, 0].min(axis=1, keepdims=True)
    per = np.diff(x[:, :, 0].min(axis=1))
    newest = (x[:, :, 17] - x[:, :, 0]) if name == "wide" else None
    older = (x[:, :, 1] - x[:, :, 17]) if name == "wide" else None
    work = x[:, :, 1] - x[:, :, 0]
    end = (x[:, :, 1] - base).max(axis=1)
    rel = (x[:, :, 2] - base).min(axis=1)
    print(f"== {name}: {sel.sum()} iterations")
    print(f"  period ns mean {per[per < 1e6].mean():.0f}")
    print(f"  work per CTA ns: mean {work.mean():.0f}, max-over-CTAs mean {work.max(1).mean():.0f}")
    if newest is not None:
        print(f"  newest loop ns: mean {newest.mean():.0f}, max {newest.max(1).mean():.0f}")
        print(f"  older work ns: mean {older.mean():.0f}, max {older.max(1).mean():.0f}")
    print(f"  start skew ns {(x[:, :, 0] - base).max(1).mean():.0f}; last work end {end.mean():.0f};"
          f" release after last end {(rel - end).mean():.0f}")
