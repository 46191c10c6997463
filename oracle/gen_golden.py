"""TEST INFRASTRUCTURE ONLY: generate tests/golden/*.npz from the UNMODIFIED reference.

Runs the reference library built by oracle/Makefile (oracle/_ref/libgeodist_ref.so,
i.e. /root/reference/proj/src compiled as-is) on small fixtures and stores its
outputs -- orderings, distances in both precisions, labels, K, relax/degenerate
counts, band traces, last_change, FPS samples/history, reorder permutations and
planar_update values -- so the GPU parity tests and the C restatement can be
checked on a box where /root/reference does not exist.

    python oracle/gen_golden.py          (from the repo root)
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def single_triangle_plus_island():
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [5, 0, 0], [6, 0, 0], [5, 1, 0]], np.float64)
    f = np.array([[0, 1, 2], [3, 4, 5]], np.int32)
    return v, f


CASES = [
    # name, mesh builder, sources, labels
    ("ico3_src0", lambda: ref.RefMesh.icosphere(3), [0], False),
    ("ico2_src0", lambda: ref.RefMesh.icosphere(2), [0], False),
    ("grid33_shear2_two", lambda: ref.RefMesh.grid(33, 33, 2.0), [0, 1088], True),
    ("grid9x5_corners", lambda: ref.RefMesh.grid(9, 5, 0.0), [0, 8], True),
    ("grid15_clumped", lambda: ref.RefMesh.grid(15, 15, 0.0), [0, 224, 112, 37], True),
    ("grid21_center", lambda: ref.RefMesh.grid(21, 21, 0.0), [220], False),
    ("strip40x6_column", lambda: ref.RefMesh.grid(40, 6, 0.0), [0, 40, 80, 120, 160, 200], True),
    ("island_src0", lambda: ref.RefMesh.from_arrays(*single_triangle_plus_island()), [0], True),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, mk, src, labels in CASES:
        R = mk()
        V, F = R.arrays()
        rec = {"vertices": V, "faces": F, "sources": np.array(src, np.int32)}
        t = R.toplesets(src)
        rec.update({"sorted": t["sorted"], "limits": t["limits"], "position": t["position"],
                    "rho": t["rho"], "unreached": t["unreached"]})
        for prec in ("single", "double"):
            r = R.ptp(src, precision=prec, labels=labels, trace=True)
            p = prec[0]
            rec[f"dist_{p}"] = r["distances"]
            rec[f"K_{p}"] = r["iterations"]
            rec[f"relax_{p}"] = r["relax_calls"]
            rec[f"degen_{p}"] = r["degenerate_calls"]
            rec[f"trace_kijU_{p}"] = r["trace"]["kijU"]
            rec[f"trace_maxrel_{p}"] = r["trace"]["max_rel"]
            rec[f"trace_conv_{p}"] = r["trace"]["converged"]
            rec[f"last_change_{p}"] = r["last_change"]
            if labels:
                rec[f"labels_{p}"] = r["labels"]
        oon, noo, pf = R.reorder(src)
        rec.update({"old_of_new": oon, "new_of_old": noo, "reordered_faces": pf})
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        print(name, R.n, "rho", t["rho"], "K", rec["K_d"], rec["K_s"])

    # farthest point sampling + voronoi
    for name, mk, m, seed in [("fps_grid17", lambda: ref.RefMesh.grid(17, 17), 8, 0),
                              ("fps_ico2", lambda: ref.RefMesh.icosphere(2), 12, 3),
                              ("fps_grid33", lambda: ref.RefMesh.grid(33, 33), 10, 0),
                              ("fps_strip30x2", lambda: ref.RefMesh.grid(30, 2), 2, 0)]:
        R = mk()
        V, F = R.arrays()
        rec = {"vertices": V, "faces": F, "m": m, "seed": seed}
        for prec in ("single", "double"):
            p = prec[0]
            r = R.fps(m, seed, precision=prec)
            rec[f"samples_{p}"] = r["samples"]
            rec[f"labels_{p}"] = r["labels"]
            rec[f"radius_{p}"] = r["radius"]
            rec[f"hist_rho_{p}"] = np.array([h["rho"] for h in r["history"]], np.int64)
            rec[f"hist_relax_{p}"] = np.array([h["relax_calls"] for h in r["history"]], np.int64)
            rec[f"hist_radius_{p}"] = np.array([h["radius"] for h in r["history"]], np.float64)
            rec[f"hist_picked_{p}"] = np.array([h["picked"] for h in r["history"]], np.int64)
            rec[f"voronoi_{p}"] = R.voronoi(r["samples"], precision=prec)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        print(name, rec["samples_d"])

    # planar_update known answers on random stars (test_update_kernel.cpp:54-83 style)
    rng = np.random.default_rng(20240817)
    cnt = 4000
    x1 = rng.uniform(-1, 1, (cnt, 3))
    x2 = rng.uniform(-1, 1, (cnt, 3))
    t1 = rng.uniform(0, 3, cnt)
    t2 = rng.uniform(0, 3, cnt)
    # edge cases: inf inputs, degenerate, rejected root, equilateral
    x1[:8] = [[1, 0, 0], [1, 0, 0], [1, 0, 0], [0, -1, 0], [1, 0, 0], [1, 0, 0], [2, 0, 0], [1, 1, 0]]
    x2[:8] = [[0.5, np.sqrt(3) / 2, 0], [0.3, 0.9, 0], [0, 1, 0], [1, -1, 0], [2, 0, 0],
              [0, 1, 0], [1, 1e-14, 0], [1, 1 + 1e-9, 0]]
    t1[:8] = [0, 0, np.inf, 0, 0.1, np.inf, 0.5, 1.0]
    t2[:8] = [0, np.inf, np.inf, 1, 0.2, 0.0, 0.25, 1.0]
    rec = {"x1": x1, "x2": x2, "t1": t1, "t2": t2}
    for prec in ("single", "double"):
        vals, sides, degs = [], [], []
        for q in range(cnt):
            v, s, d = ref.planar(x1[q], x2[q], t1[q], t2[q], single=prec == "single")
            vals.append(v)
            sides.append(s)
            degs.append(d)
        rec[f"value_{prec[0]}"] = np.array(vals)
        rec[f"side_{prec[0]}"] = np.array(sides, np.int32)
        rec[f"degen_{prec[0]}"] = np.array(degs, bool)
    np.savez_compressed(os.path.join(OUT, "planar_update.npz"), **rec)
    print("planar_update", cnt)
    acceptance()


def acceptance():
    """Reference acceptance-suite output (timings stripped): oracle/_ref/acceptance_ref."""
    import re
    import subprocess
    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")
    out = subprocess.run([exe], capture_output=True, text=True).stdout
    text = "".join(re.sub(r" \[[0-9.]+s\]$", "", ln) + "\n" for ln in out.splitlines())
    open(os.path.join(OUT, "acceptance_reference.txt"), "w").write(text)


if __name__ == "__main__":
    main()

