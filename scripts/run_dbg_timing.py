"""Run one field with per-iteration CTA timestamps (GEODIST_DEBUG_TIMING) and summarise.

  python scripts/run_dbg_timing.py [single|double] [ico8|torus|grid1001]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GEODIST_DEBUG_TIMING"] = "2000"
import paper_1810_08218_b200 as g  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "single"
mesh = sys.argv[2] if len(sys.argv) > 2 else "ico8"
if mesh == "torus":
    M = g.generate_torus(1000, 1000)
elif mesh == "grid1001":
    M = g.generate_grid(1001, 1001)
else:
    v, f = g.noisy_icosphere_arrays(8, 2e-3, 1)
    M = g.Mesh(v, f)
src = [500 * 1001 + 500] if mesh == "grid1001" else [0]
os.makedirs("gpurun_out", exist_ok=True)
for _ in range(2):
    r = g.geodesics(M, src, precision=prec)
print("K", r["iterations"], "device ms", 1e3 * r["device_seconds"])
subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "dbg_timing_summary.py"),
                "gpurun_out/dbg_timing.bin"])
