#!/usr/bin/env python
"""Benchmark: ms per single-source PTP distance field on a 1M-vertex mesh, one B200.

Workloads (--workload; SURVEY §8d pins every input):
  torus1000 (default)  the metric's configuration: 1000x1000 torus (R=3, r=1,
                       1,000,000 vertices, 2,000,000 faces; BASELINE configs 4/5),
                       single source {0}
  grid1001             the paper's 1001^2 grid (1,002,001 vertices), centre source
  icosphere8           noise-perturbed icosphere subdiv-8 (655,362 vertices, sigma =
                       2e-3, std::mt19937(1)), source {0} (BASELINE configs[1])
  batch512             BASELINE configs[4]: 512 single-source queries s_q = q*floor(n/512)
                       on the 1000^2 torus, sharded over the ranks (batch.run_sharded:
                       per-GPU concurrent query groups, NCCL gather to rank 0 inside
                       the timed region); a step = the whole 512-query batch

A step of a single-field workload is one complete distance field: fused
on-device toplesets BFS + banded Jacobi relaxation to convergence + copy-out.
With N GPUs (torchrun, one rank per GPU) every rank computes one independent
field per step -- rank r, step s solves source (s*N + r) * floor(nu/64) on the
torus's outer equator row (rotations of source 0: equal work per field; N = 1
is source 0 every step) -- and the fields are gathered to rank 0 over NCCL
inside the timed region (weak scaling, the only collective).

  value  : device time (CUDA events on the launching stream) per field, inputs
           resident in HBM, L2 flushed between steps; whole-job ms per field =
           max-over-ranks time / (fields all ranks solved)
  e2e    : the same field through the public API geodesics() with host
           buffers: source upload + float64 distance download every step
  roofline: SURVEY §8(d) byte model (fp32 12U+16C / fp64 20U+28C bytes per
           field) over the solver's device time against MEASURED_PEAKS.json
           hbm_gbs; roofline.l2 from the committed ncu capture of the same field
           against the L2 read bandwidth measured on the box (profiles/round2)
  cpu_baseline: the unmodified reference (oracle/_ref, OpenMP, all host
           threads) on one field of the same workload, rank 0 only

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision single|double]
                  [--workload torus1000|grid1001|icosphere8|batch512]
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
METRIC = "ms per distance field @1M verts"
# SURVEY §8d inputs
TORUS = dict(nu=1000, nv=1000, R=3.0, r=1.0)
GRID = 1001
SIGMA, SUBDIV = 2e-3, 8
NQ_BATCH = 512
EPS = 1e-3
# the reference arm stops adding timed fields after this much CPU time (>= 1 field)
REF_BUDGET_S = 90.0

WORKLOADS = {
    "torus1000": "1000x1000 torus R=3 r=1 (1,000,000 vertices), single source {0} "
                 "(SURVEY 8d; BASELINE configs 4/5 mesh)",
    "grid1001": "paper grid 1001x1001 (1,002,001 vertices), centre source {501000}",
    "icosphere8": "noisy icosphere subdiv-8 sigma=2e-3 mt19937(1) (655,362 vertices), "
                  "source {0} (BASELINE configs[1])",
    "batch512": "512 single-source queries s_q = q*floor(n/512) on the 1000x1000 torus "
                "(BASELINE configs[4]), sharded over the ranks",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def ncu_summary(workload, precision):
    """The committed ncu --set full summary of this workload's field (profiles/round2)."""
    path = os.path.join(ROOT, "profiles", "round2", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(f"{workload}_{precision}")
    except Exception:
        return None


def l2_peak():
    path = os.path.join(ROOT, "profiles", "round2", "l2_peak.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["l2_read_gbs"])
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


def product_arrays(workload):
    """Our arm's input mesh (the product's generators)."""
    import paper_1810_08218_b200 as g
    if workload in ("torus1000", "batch512"):
        return g.torus_arrays(TORUS["nu"], TORUS["nv"], TORUS["R"], TORUS["r"])
    if workload == "grid1001":
        return g.grid_arrays(GRID, GRID, 0.0)
    return g.noisy_icosphere_arrays(SUBDIV, SIGMA, 1)


def reference_mesh(workload):
    """The reference arm's input mesh, built on the reference's own types by
    oracle/ref_capi.cpp (bit-identical to product_arrays: tests/test_capi_host.py);
    the product library is never loaded on this arm."""
    from oracle import ref
    if workload in ("torus1000", "batch512"):
        return ref.RefMesh.torus(TORUS["nu"], TORUS["nv"], TORUS["R"], TORUS["r"])
    if workload == "grid1001":
        return ref.RefMesh.grid(GRID, GRID, 0.0)
    return ref.RefMesh.noisy_icosphere(SUBDIV, SIGMA, 1)


def field_source(workload, rank, step, world):
    """Source of rank `rank`'s field at `step`.  N = 1: the workload's pinned source every
    step.  N > 1 (torus): rotations of source 0 along the outer equator row (j = 0), so
    every rank's field is the same amount of work (weak scaling)."""
    if workload == "grid1001":
        return (GRID // 2) * GRID + GRID // 2
    if world == 1 or workload != "torus1000":
        return 0
    return ((step * world + rank) * (TORUS["nu"] // 64)) % TORUS["nu"]


def batch_queries(n):
    step = max(1, n // NQ_BATCH)
    return [[q * step] for q in range(NQ_BATCH)]


def config_block(workload, n, precision, nranks, fields_per_step):
    return {"workload": WORKLOADS[workload], "name": workload, "n_vertices": n,
            "sources_per_field": 1, "fields_per_step": fields_per_step,
            "precision": precision, "epsilon": EPS,
            "l2": "flushed between timed steps (persisting lines demoted, then a 256 MiB write)",
            "solver": "v4 ptp_run4_kernel (narrow/wide instantiations)",
            "parallelism": f"independent fields, {nranks} rank(s), NCCL gather to rank 0"}


def host_threads():
    """All host threads this process may run on.  (torchrun exports OMP_NUM_THREADS=1, so
    the reference's 'workers = 0 -> omp_get_max_threads()' would run it on one thread.)"""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    """The reference arm: the unmodified reference (oracle/_ref) on the box's host cores,
    same workload, metric and unit; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    R = reference_mesh(args.workload)
    n = R.n
    srcs = [q[0] for q in batch_queries(n)] if args.workload == "batch512" else None
    # untimed warm-up fields (page in the library, the mesh and the OpenMP team), at most
    # args.warmup and at most ~20 s of CPU work
    warm, w0 = 0, time.perf_counter()
    for s in range(args.warmup):
        src = srcs[-1 - s] if srcs else field_source(args.workload, 0, 1000 + s, 1)
        R.ptp([src], precision=args.precision, workers=host_threads())
        warm += 1
        if time.perf_counter() - w0 > 20.0:
            break
    times, started, r = [], time.perf_counter(), None
    for s in range(args.steps):
        src = srcs[s % len(srcs)] if srcs else field_source(args.workload, 0, s, 1)
        r = R.ptp([src], precision=args.precision, workers=host_threads())
        times.append(r["wall_seconds"] + r["toplesets_seconds"])
        if time.perf_counter() - started > REF_BUDGET_S:
            break
    ms = 1e3 * sum(times) / len(times)
    cores = int(r["workers"])
    sample = (f"{len(times)} of {args.steps} requested fields (stops after {REF_BUDGET_S:.0f} s "
              "of CPU work), compute_toplesets + ptp_run with the reference's own timers, "
              f"unmodified reference (oracle/_ref), OpenMP on all host threads; {warm} untimed "
              "warm-up field(s)")
    if srcs:
        sample += f"; queries 0..{len(times) - 1} of the 512-query list (prefix, per field)"
    line = {"metric": METRIC, "value": ms, "unit": "ms",
            "n_gpus": args.gpus, "steps": len(times), "warmup": warm, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "single" else "f64", "data": "synthetic",
            "config": config_block(args.workload, n, args.precision, 1, 1), "impl": "reference",
            "iterations": r["iterations"],
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def cpu_baseline_field(workload, precision, src):
    """One field of the unmodified reference (oracle/_ref), all host threads."""
    R = reference_mesh(workload)
    return R.ptp([src], precision=precision, workers=host_threads())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", default="single", choices=["single", "double"])
    ap.add_argument("--workload", default="torus1000", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_1810_08218_b200 as g
    from paper_1810_08218_b200 import batch

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

    V, F = product_arrays(args.workload)
    n = len(V)
    mesh = g.Mesh(V, F, device=local)
    tdtype = torch.float32 if args.precision == "single" else torch.float64
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def flush_l2():
        """evict L2 between timed steps: the solver's persisting lines are demoted first,
        then a 256 MiB write (2x the L2) replaces every line"""
        g.lib().geodist_reset_persisting_l2()
        flush.zero_()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def gather_dev(t):
        """results of every rank to rank 0 (the only collective), device-timed"""
        if world == 1:
            return 0.0
        src = t if backend == "nccl" else t.cpu()
        got = [torch.empty_like(src) for _ in range(world)] if rank == 0 else None
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        dist.gather(src, got, dst=0)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if backend != "nccl":
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    is_batch = args.workload == "batch512"
    queries = batch_queries(n) if is_batch else None
    # warm-up (also packs the geometry tables once and sizes the workspaces)
    if is_batch:
        for s in range(args.warmup if args.warmup <= 1 else 1):
            batch.run_sharded(mesh, queries[:8 * world], precision=args.precision)
    else:
        scratch = torch.empty((1, n), dtype=tdtype, device="cuda")
        for s in range(args.warmup):
            g.batch_geodesics_device(mesh, [[field_source(args.workload, rank, s + 1000, world)]],
                                     scratch[0].data_ptr(), precision=args.precision)

    launches0 = g._capi.kernel_launches()
    dev_s, stats, fields_done = [], [], 0
    steps = args.steps if not is_batch else max(1, min(args.steps, 2))
    results = None
    barrier()
    with Clocks(local) as clk:
        for s in range(steps):
            flush_l2()
            torch.cuda.synchronize()
            if is_batch:
                # the whole 512-query list per step: device time of the per-GPU batch
                # launches plus the NCCL gather
                t0 = torch.cuda.Event(enable_timing=True)
                t1 = torch.cuda.Event(enable_timing=True)
                t0.record()
                fields, st = batch.run_sharded(mesh, queries, precision=args.precision)
                t1.record()
                torch.cuda.synchronize()
                dev_s.append(t0.elapsed_time(t1) * 1e-3)
                stats.extend(st)
                fields_done += len(queries)
                results = fields
            else:
                if results is None:
                    results = torch.empty((steps, n), dtype=tdtype, device="cuda")
                st = g.batch_geodesics_device(
                    mesh, [[field_source(args.workload, rank, s, world)]],
                    results[s].data_ptr(), precision=args.precision)[0]
                dev_s.append(st["device_seconds"])
                stats.append(st)
                fields_done += world
        if not is_batch:
            dev_s.append(gather_dev(results))
        barrier()
    launches = g._capi.kernel_launches() - launches0
    total = max_over_ranks(sum(dev_s))
    ms_field = 1e3 * total / fields_done
    ms_step = 1e3 * total / steps

    # end to end through the public API (host buffers, H2D source + D2H distances)
    e2e_ms = None
    if not is_batch:
        e2e_s = []
        out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        for s in range(args.warmup):  # untimed: first calls size the API's device buffers
            g.geodesics(mesh, [field_source(args.workload, rank, s + 1000, world)],
                        precision=args.precision, out=out)
        barrier()
        for s in range(steps):
            flush_l2()
            torch.cuda.synchronize()
            t = time.perf_counter()
            g.geodesics(mesh, [field_source(args.workload, rank, s, world)],
                        precision=args.precision, out=out)
            e2e_s.append(time.perf_counter() - t)
        barrier()
        e2e_ms = 1e3 * max_over_ranks(sum(e2e_s)) / (world * steps)

    if rank == 0:
        U = sum(x["vertex_updates"] for x in stats)
        Cc = sum(x["relax_calls"] for x in stats)
        a, b = (12, 16) if args.precision == "single" else (20, 28)
        byts = a * U + b * Cc
        kernel_s = sum(dev_s[:steps])
        peak, peak_kind = peaks()
        achieved = byts / kernel_s / 1e9
        nfield = len(stats)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_kind,
                "byte_model": f"{a}*U + {b}*C per field (SURVEY 8d)",
                "algorithmic_bytes_per_field": byts / nfield,
                "kernel": "ptp_run4_kernel (all launches of a field: narrow + wide "
                          "instantiations), CUDA events on the solver's stream"}
        summ = ncu_summary(args.workload, args.precision)
        if summ:
            roof["traffic"] = summ.get("dram_bytes_per_field")
            roof["traffic_source"] = "profiles/round2/ncu_summary.json (ncu --set full, same field)"
            l2p = l2_peak()
            if l2p and summ.get("l2_bytes_per_field"):
                ach = summ["l2_bytes_per_field"] / (summ["duration_ns_per_field"] * 1e-9) / 1e9
                roof["l2"] = {"achieved": ach, "peak": l2p, "unit": "GB/s", "frac": ach / l2p,
                              "sectors_per_request": summ.get("l2_sectors_per_request"),
                              "source": "ncu lts__t_sectors x 32 B over the field's solver "
                                        "time; peak = profiles/round2/l2_peak.json"}
        line = {
            "metric": METRIC, "value": ms_field, "unit": "ms",
            "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "single" else "f64", "data": "synthetic",
            "config": config_block(args.workload, n, args.precision, world,
                                   len(queries) if is_batch else world),
            "roofline": roof,
            "vertex_updates_per_s": U / kernel_s,
            "iterations": [x["iterations"] for x in stats][:3],
            "rho": stats[0]["rho"], "U_per_field": U / nfield, "C_per_field": Cc / nfield,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if is_batch:
            # the same queries one field at a time on the whole GPU (every 16th source,
            # untimed by the step clock): what batching buys per query
            sample = queries[::16]
            scratch = torch.empty((1, n), dtype=tdtype, device="cuda")
            one = [g.batch_geodesics_device(mesh, [q], scratch[0].data_ptr(),
                                            precision=args.precision)[0] for q in sample]
            per_one = 1e3 * sum(x["device_seconds"] for x in one) / len(one)
            u_one = sum(x["vertex_updates"] for x in one) / len(one)
            line["vs_single_fields"] = {
                "batched_ms_per_query": ms_field, "one_at_a_time_ms_per_query": per_one,
                "sample": f"{len(sample)} of the {len(queries)} sources (every 16th), one "
                          "field per launch sequence on the whole GPU, device time",
                "U_per_query_sample": u_one}
        if e2e_ms is not None:
            line["e2e"] = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 4,
                           "d2h_bytes_per_step": 8 * n,
                           "api": "paper_1810_08218_b200.geodesics",
                           "host_buffers": "source list in host memory, float64 distances "
                                           "into a pinned host array"}
        if not args.no_cpu_baseline and world == 1 and not is_batch:
            try:
                from oracle import ref
                if ref.available():
                    src = field_source(args.workload, 0, 0, 1)
                    r = cpu_baseline_field(args.workload, args.precision, src)
                    mine = results[0].double().cpu().numpy()
                    same = np.array_equal(mine.view(np.int64), r["distances"].view(np.int64))
                    line["cpu_baseline"] = {
                        "value": 1e3 * (r["wall_seconds"] + r["toplesets_seconds"]), "unit": "ms",
                        "cores": int(r["workers"]), "kind": "reference",
                        "sample": f"1 field, source {src} (compute_toplesets + ptp_run, "
                                  "reference timers), unmodified reference built by "
                                  "oracle/Makefile",
                        "ptp_run_ms": 1e3 * r["wall_seconds"],
                        "iterations": r["iterations"]}
                    line["parity"] = {"vs": f"reference {args.precision}_fp, source {src}",
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
