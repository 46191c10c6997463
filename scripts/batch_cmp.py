"""Batched queries vs the same queries one field at a time (device time per query).

  python scripts/batch_cmp.py [single|double] [count]   (sources: every 16th of the 512
  BASELINE configs[4] queries s_q = q*floor(n/512) on the 1000^2 torus)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1810_08218_b200 as g  # noqa: E402
from paper_1810_08218_b200 import batch  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "single"
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 32
M = g.generate_torus(1000, 1000)
n = M.n_vertices
qs = batch.even_sources(n, 512)[::512 // cnt][:cnt]
dt = torch.float32 if prec == "single" else torch.float64
out = torch.empty((len(qs), n), dtype=dt, device="cuda")
res = {}
g.batch_geodesics_device(M, qs[:2], out.data_ptr(), precision=prec, groups=1)  # warm-up
one = [g.batch_geodesics_device(M, [q], out[i].data_ptr(), precision=prec)[0]
       for i, q in enumerate(qs)]
res["one_at_a_time_ms_per_query"] = 1e3 * sum(x["device_seconds"] for x in one) / len(qs)
res["U_per_query"] = sum(x["vertex_updates"] for x in one) / len(qs)
ref = out.clone()
for groups in (1, 2, 4, 8, 0):
    st = g.batch_geodesics_device(M, qs, out.data_ptr(), precision=prec, groups=groups)
    res[f"groups{groups}_ms_per_query"] = 1e3 * st[0]["device_seconds"] / len(qs)  # whole batch
    res[f"groups{groups}_equal"] = bool(torch.equal(out, ref))
print(json.dumps(res, indent=1))
