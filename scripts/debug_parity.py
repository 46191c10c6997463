"""Compare the GPU trace/distances with a golden case and report the first divergence."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import golden, bits
import paper_1810_08218_b200 as g

name = sys.argv[1]
prec = sys.argv[2] if len(sys.argv) > 2 else "single"
gd = golden(name)
M = g.Mesh(gd["vertices"], gd["faces"])
p = prec[0]
labels = f"labels_{p}" in gd
r = g.geodesics(M, gd["sources"], precision=prec, labels=labels, trace=True)
tr = np.array([[t["k"], t["i"], t["j"], t["updated"]] for t in r["trace"]])
gt = gd[f"trace_kijU_{p}"]
print("K gpu", r["iterations"], "ref", int(gd[f"K_{p}"]), "rho", r["rho"], int(gd["rho"]))
n = min(len(tr), len(gt))
bad = np.nonzero((tr[:n] != gt[:n]).any(1))[0]
if len(bad):
    q = bad[0]
    print("first trace row mismatch at", q, "gpu", tr[q], "ref", gt[q])
mr = np.array([t["max_rel_change"] for t in r["trace"]])
bm = np.nonzero(bits(mr[:n]) != bits(gd[f"trace_maxrel_{p}"][:n]))[0]
if len(bm):
    q = bm[0]
    print("first max_rel mismatch at", q, mr[q], gd[f"trace_maxrel_{p}"][q])
dd = np.nonzero(bits(r["distances"]) != bits(gd[f"dist_{p}"]))[0]
print("distance mismatches", len(dd), dd[:10], r["distances"][dd[:5]], gd[f"dist_{p}"][dd[:5]])
t = g.toplesets(M, gd["sources"])
print("toplesets exact:", np.array_equal(t["sorted"], gd["sorted"]))
