#!/usr/bin/env python
"""Benchmark: ms per single-source PTP distance field on a B200.

Workload (BASELINE.json configs[1]): noise-perturbed icosphere subdiv-8
(655,362 vertices, radial noise sigma = 2e-3, std::mt19937(1)), one source per
field.  A step is one complete distance field: fused on-device toplesets BFS +
banded Jacobi relaxation to convergence + copy-out.  N GPUs (torchrun, one rank
per GPU) each compute independent fields (weak scaling; the per-query results
are gathered to rank 0 over NCCL at the end of the timed region).

  value  : device time (CUDA events on the launching stream) per field, inputs
           resident in HBM, L2 flushed between steps, summed over the K steps;
           whole-job ms per field = max-over-ranks time / (N * K)
  e2e    : the same field through the public API geodesics() with host
           buffers: source upload + distance download (float64) every step
  roofline: SURVEY §8(d) byte model, fp32 12U+16C / fp64 20U+28C bytes per
           field, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline: the unmodified reference (oracle/_ref, OpenMP, all host
           threads) on one field of the same workload, rank 0 only

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision single|double]
  python bench.py --impl reference ...   (reference CPU path, rank 0 only)
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0
SIGMA = 2e-3
SUBDIV = 8


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def ncu_traffic(precision):
    """dram read+write bytes per launch of the run kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            s = json.load(fh)
        return s.get(f"ptp_run_kernel_{precision}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class Clocks:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, device):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def workload_arrays():
    import paper_1810_08218_b200 as g
    return g.noisy_icosphere_arrays(SUBDIV, SIGMA, 1)


def source_for(rank, step, n):
    return 0  # the BASELINE config: single source {0}, every rank and step


def config_block(n, precision, nranks):
    return {"workload": "noisy icosphere subdiv-8 single-source distance field (BASELINE configs[1])",
            "n_vertices": n, "noise_sigma": SIGMA, "noise_rng": "std::mt19937(1) normal",
            "sources_per_field": 1, "precision": precision, "epsilon": 1e-3,
            "l2": "flushed (256 MiB write) between timed steps",
            "solver": {"2": "v2 ptp_run_kernel", "3": "v3 ptp_run3_kernel"}.get(
                os.environ.get("GEODIST_SOLVER", "4")[:1], "v4 ptp_run4_kernel"),
            "parallelism": f"independent fields, {nranks} rank(s)"}


def host_threads():
    """All host threads this process may run on.  (torchrun exports OMP_NUM_THREADS=1, so
    the reference's 'workers = 0 -> omp_get_max_threads()' would run it on one thread.)"""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_field(V, F, precision, src=0):
    """One field on the unmodified reference (oracle/_ref), all host threads."""
    from oracle import ref
    R = ref.RefMesh.from_arrays(V, F)
    r = R.ptp([src], precision=precision, workers=host_threads())
    return R, r


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    V, F = workload_arrays()
    R = ref.RefMesh.from_arrays(V, F)
    times = []
    for s in range(args.warmup + args.steps):
        r = R.ptp([source_for(0, s, len(V))], precision=args.precision, workers=host_threads())
        if s >= args.warmup:
            times.append(r["wall_seconds"] + r["toplesets_seconds"])
    ms = 1e3 * sum(times) / len(times)
    cores = int(r["workers"])
    line = {"metric": "ms per distance field @1M verts", "value": ms, "unit": "ms",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "single" else "f64", "data": "synthetic",
            "config": config_block(len(V), args.precision, 1), "impl": "reference",
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "reference",
                             "sample": f"{args.steps} fields (compute_toplesets + ptp_run, "
                                       "reference's own timers), unmodified reference, OpenMP"},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", default="single", choices=["single", "double"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_1810_08218_b200 as g

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks for the multi-rank path on a one-GPU box: every rank on one device,
    # gloo instead of NCCL (collectives then run on host copies)
    if os.environ.get("BENCH_FORCE_DEVICE"):
        local = int(os.environ["BENCH_FORCE_DEVICE"])
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def coll(t):  # tensor as the process group's backend wants it
        return t if backend == "nccl" else t.cpu()

    V, F = workload_arrays()
    n = len(V)
    mesh = g.Mesh(V, F, device=local)
    tdtype = torch.float32 if args.precision == "single" else torch.float64
    results = torch.empty((args.steps, n), dtype=tdtype, device="cuda")
    scratch = torch.empty((args.warmup, n), dtype=tdtype, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also packs the geometry tables once)
    for s in range(args.warmup):
        g.batch_geodesics_device(mesh, [[source_for(rank, s + 1000, n)]],
                                 scratch[s].data_ptr(), precision=args.precision)

    launches0 = g._capi.kernel_launches()
    dev_s, stats = [], []
    barrier()
    with Clocks(local) as clk:
        for s in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            st = g.batch_geodesics_device(mesh, [[source_for(rank, s, n)]], results[s].data_ptr(),
                                          precision=args.precision)[0]
            dev_s.append(st["device_seconds"])
            stats.append(st)
        if world > 1:
            # per-query results gathered to rank 0 (the only collective: SURVEY 8e)
            res = coll(results)
            gathered = [torch.empty_like(res) for _ in range(world)] if rank == 0 else None
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            dist.gather(res, gathered, dst=0)
            t1.record()
            torch.cuda.synchronize()
            dev_s.append(t0.elapsed_time(t1) * 1e-3)
        barrier()
    launches = g._capi.kernel_launches() - launches0
    total = sum(dev_s)
    if world > 1:
        tt = coll(torch.tensor([total], dtype=torch.float64, device="cuda"))
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    ms_field = 1e3 * total / (world * args.steps)
    ms_step = 1e3 * total / args.steps

    # end to end through the public API (host buffers, H2D source + D2H distances)
    e2e_s = []
    # result lands in pinned host memory (the D2H copy runs at full PCIe/C2C speed)
    out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    for s in range(args.warmup):  # untimed: first calls size the API's device buffers
        g.geodesics(mesh, [source_for(rank, s + 1000, n)], precision=args.precision, out=out)
    barrier()
    for s in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        g.geodesics(mesh, [source_for(rank, s, n)], precision=args.precision, out=out)
        e2e_s.append(time.perf_counter() - t)
    barrier()
    e2e_total = sum(e2e_s)
    if world > 1:
        tt = coll(torch.tensor([e2e_total], dtype=torch.float64, device="cuda"))
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_total = float(tt.item())
    e2e_ms = 1e3 * e2e_total / (world * args.steps)

    if rank == 0:
        U = sum(x["vertex_updates"] for x in stats)
        Cc = sum(x["relax_calls"] for x in stats)
        a, b = (12, 16) if args.precision == "single" else (20, 28)
        byts = a * U + b * Cc
        kernel_s = sum(dev_s[:args.steps])
        peak, peak_kind = peaks()
        achieved = byts / kernel_s / 1e9
        line = {
            "metric": "ms per distance field @1M verts", "value": ms_field, "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "single" else "f64", "data": "synthetic",
            "config": config_block(n, args.precision, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.precision),
                         "peak_source": peak_kind,
                         "byte_model": f"{a}*U + {b}*C per field (SURVEY 8d)",
                         "algorithmic_bytes_per_field": byts / args.steps},
            "vertex_updates_per_s": U / kernel_s,
            "iterations": [x["iterations"] for x in stats][:3],
            "rho": stats[0]["rho"], "U_per_field": U / args.steps, "C_per_field": Cc / args.steps,
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 4,
                    "d2h_bytes_per_step": 8 * n, "api": "paper_1810_08218_b200.geodesics",
                    "host_buffers": "source list in host memory, float64 distances into a "
                                    "pinned host array"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline and world == 1:
            try:
                from oracle import ref
                if ref.available():
                    R, r = cpu_reference_field(V, F, args.precision, 0)
                    mine = results[0].double().cpu().numpy()
                    same = np.array_equal(mine.view(np.int64), r["distances"].view(np.int64))
                    line["cpu_baseline"] = {
                        "value": 1e3 * (r["wall_seconds"] + r["toplesets_seconds"]), "unit": "ms",
                        "cores": int(r["workers"]), "kind": "reference",
                        "sample": "1 field, source 0 (compute_toplesets + ptp_run, reference "
                                  "timers), unmodified reference built by oracle/Makefile",
                        "ptp_run_ms": 1e3 * r["wall_seconds"],
                        "iterations": r["iterations"]}
                    line["parity"] = {"vs": f"reference {args.precision}_fp, source 0",
                                      "bit_exact": bool(same),
                                      "iterations_gpu": stats[0]["iterations"],
                                      "iterations_ref": r["iterations"]}
            except Exception as e:  # the baseline must never break the bench line
                line["cpu_baseline"] = {"error": str(e)[:200]}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
