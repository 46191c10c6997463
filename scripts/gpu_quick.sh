#!/bin/bash
# Quick GPU check: full parity suite, corner microbenchmark, v4 timing + bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 60 build/microbench_corner
GEODIST_SOLVER=4 timeout 120 python scripts/run_dbg_timing.py > gpurun_out/dbg_v4.txt 2>&1; head -16 gpurun_out/dbg_v4.txt
for V in 2 4; do GEODIST_SOLVER=$V timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_v$V.json 2> gpurun_out/bench_v$V.err; echo "v$V"; cut -c1-120 gpurun_out/bench_v$V.json; done
