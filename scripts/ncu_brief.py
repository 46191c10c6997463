"""Headline counters of an ncu report: time, instructions, lane efficiency, L2/DRAM
traffic, issue, occupancy and the top stall reasons.

    python scripts/ncu_brief.py gpurun_out/prof.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("smsp__inst_executed.sum", "warp_inst"),
        ("sass__thread_inst_executed_true_per_opcode", "thread_inst"),
        ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_rd_sectors"),
        ("lts__t_sectors_srcunit_tex_op_write.sum", "l2_wr_sectors"),
        ("lts__t_requests_srcunit_tex_op_read.sum", "l2_rd_requests"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_thru%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
        ("launch__registers_per_thread", "regs")]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {a: (b, c) for a, b, c in zip(rows[0], rows[1], rows[2])}


for rep in sys.argv[1:]:
    d = load(rep)
    print("==", rep)
    for k, name in KEYS:
        if k in d:
            print(f"  {name:14s} {d[k][1]} {d[k][0]}")
    try:
        wi = float(d["smsp__inst_executed.sum"][1].replace(",", ""))
        ti = float(d["sass__thread_inst_executed_true_per_opcode"][1].replace(",", ""))
        rs = float(d["lts__t_sectors_srcunit_tex_op_read.sum"][1].replace(",", ""))
        rq = float(d["lts__t_requests_srcunit_tex_op_read.sum"][1].replace(",", ""))
        print(f"  lane_eff       {ti / wi / 32:.3f}   l2 sectors/request {rs / rq:.2f}")
    except (KeyError, ValueError, ZeroDivisionError):
        pass
    st = [(k, d[k][1]) for k in d if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:7]
    print("  stalls/issue  " + "  ".join(
        f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={float(v):.2f}"
        for k, v in st))
