"""Repro for the batched v4 path (several queries per group, labels)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_08218_b200 as g
v, f = g.noisy_icosphere_arrays(5, 2e-3, 1)
M = g.Mesh(v, f)
queries = [[q * 97] for q in range(9)] + [[3, 5000, 9000]]
for prec in ("single", "double"):
    for groups in (1, 3, 4):
        out = g.batch_geodesics(M, queries, precision=prec, labels=True, groups=groups)
        bad = 0
        for q, src in enumerate(queries):
            one = g.geodesics(M, src, precision=prec, labels=True)
            bad += not np.array_equal(out["distances"][q], one["distances"])
        print(prec, groups, "mismatching queries:", bad, flush=True)
