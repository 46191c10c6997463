#!/bin/bash
# Quick GPU check: v4 parity suite, v4 per-iteration timing, ico8 bench (both precisions).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "v4" > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 120 python scripts/run_dbg_timing.py single ico8 > gpurun_out/dbg_v4.txt 2>&1; head -16 gpurun_out/dbg_v4.txt
for P in single double; do timeout 300 python bench.py --steps 10 --no-cpu-baseline --precision $P > gpurun_out/bench_$P.json 2> gpurun_out/bench_$P.err; cut -c1-110 gpurun_out/bench_$P.json; done
