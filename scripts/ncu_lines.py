"""Per-source-line instruction and stall-sample totals from an ncu report
(--page source --print-source cuda,sass): where a kernel's issue slots and stalls go.

    python scripts/ncu_lines.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
f = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        rows.append((f, int(r[0]), r[1].strip()[:90], int(r[4]), int(r[7]), int(r[8])))
    except (ValueError, IndexError):
        pass
tot_i = sum(x[4] for x in rows) or 1
tot_s = sum(x[3] for x in rows) or 1
print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
print("  inst%  stall%  file:line  source")
for x in sorted(rows, key=lambda x: -(x[4] / tot_i + x[3] / tot_s))[:top]:
    print(f"{100 * x[4] / tot_i:6.2f} {100 * x[3] / tot_s:6.2f}  {x[0]}:{x[1]}  {x[2]}")
