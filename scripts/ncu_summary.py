"""Summarise ncu reports of the solver kernel into profiles/ (JSON + markdown).

    python scripts/ncu_summary.py gpurun_out/prof_single.ncu-rep gpurun_out/prof_double.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
    "lts__t_sectors_srcunit_tex_op_write.sum": "l2_write_sectors",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__func_cache_config": "func_cache_config",
}
UNITS = {"dram_read": None, "dram_write": None, "l2_bytes": None}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def to_bytes(u, v):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}.get(u, 1)
    return v * scale


def summarise(rep):
    r = raw(rep)
    s = {"report": os.path.basename(rep)}
    for k, name in WANT.items():
        if k in r:
            u, v = r[k]
            if name in UNITS:
                s[name] = to_bytes(u, v)
            elif name == "duration_ns":
                s[name] = float(v.replace(",", "")) * {"msecond": 1e6, "ms": 1e6, "us": 1e3, "ns": 1.0, "usecond": 1e3,
                                                       "nsecond": 1.0, "second": 1e9}.get(u, 1.0)
            else:
                try:
                    s[name] = float(v.replace(",", ""))
                except ValueError:
                    s[name] = v
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[1].replace(",", ""))
              for k, v in r.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    s["stall_pct"] = {k: round(100 * v / tot, 1)
                      for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
    if "dram_read" in s:
        s["dram_bytes_per_launch"] = s["dram_read"] + s.get("dram_write", 0.0)
    return s


def main():
    out = {}
    for rep in sys.argv[1:]:
        base = os.path.basename(rep).replace(".ncu-rep", "")
        if "torus" in base:
            key = "torus_" + ("double" if "double" in base else "single")
        else:
            key = "ptp_run_kernel_" + ("double" if "double" in base else "single")
        out[key] = summarise(rep)
        out[key]["kernel"] = "ptp_run4_kernel (v4)"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    old = {}
    if os.path.exists(path):
        old = json.load(open(path))
    old.update(out)
    json.dump(old, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
