#!/bin/bash
# v4 bring-up: parity tests on the v4 path, timing of one ico8 field per solver.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "v4" > gpurun_out/pytest_v4.txt 2>&1; tail -15 gpurun_out/pytest_v4.txt
for V in 4; do
  GEODIST_SOLVER=$V timeout 120 python scripts/run_dbg_timing.py > gpurun_out/dbg_v$V.txt 2>&1; head -16 gpurun_out/dbg_v$V.txt
done
GEODIST_SOLVER=4 timeout 300 python bench.py --steps 10 > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err; cut -c1-300 gpurun_out/bench_v4.json; tail -3 gpurun_out/bench_v4.err
