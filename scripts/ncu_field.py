"""Field-level ncu counters for bench.py's roofline (profiles/round2/ncu_summary.json).

On the GPU box (one process per workload):
    ncu --metrics <METRICS> --clock-control none -k regex:ptp_run4 --csv \
        --log-file gpurun_out/field_<w>_<p>.csv python scripts/one_field.py <w> <p>
Here:
    python scripts/ncu_field.py gpurun_out/field_*.csv  -> profiles/round2/ncu_summary.json

one_field.py solves the same field twice; the second field's solver launches (the
narrow / wide instantiations) are summed: DRAM bytes, L2 sectors and requests,
duration.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,"
           "lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors.sum")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6, "second": 1e9}


def launches(path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per = {}
    for r in rows:
        lid = int(r["ID"])
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1)
        per.setdefault(lid, {"kernel": r["Kernel Name"]})[r["Metric Name"]] = v
    return [per[k] for k in sorted(per)]


def main(paths):
    out_path = os.path.join(ROOT, "profiles", "round2", "ncu_summary.json")
    summary = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for p in paths:
        name = os.path.basename(p)[len("field_"):-len(".csv")]
        ls = [x for x in launches(p) if "ptp_run4" in x["kernel"]]
        half = ls[len(ls) // 2:]  # the second of the two identical fields
        tot = lambda k: sum(x.get(k, 0.0) for x in half)
        sect = tot("lts__t_sectors.sum")
        rd_s = tot("lts__t_sectors_srcunit_tex_op_read.sum")
        rq = tot("lts__t_requests_srcunit_tex_op_read.sum")
        summary[name] = {
            "launches": len(half), "kernels": sorted({x["kernel"][:60] for x in half}),
            "duration_ns_per_field": tot("gpu__time_duration.sum"),
            "dram_bytes_per_field": tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum"),
            # data traffic from the SMs (loads + stores); lts__t_sectors also counts the
            # barrier word's polls and atomics
            "l2_bytes_per_field": 32.0 * (rd_s + tot("lts__t_sectors_srcunit_tex_op_write.sum")),
            "l2_all_sectors_bytes_per_field": 32.0 * sect,
            "l2_read_sectors": rd_s, "l2_read_requests": rq,
            "l2_sectors_per_request": rd_s / rq if rq else None,
            "source": os.path.basename(p) + " (ncu --metrics, --clock-control none; cold-cache, "
                      "serialised replays)"}
    with open(out_path, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
