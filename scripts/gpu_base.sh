#!/bin/bash
# baseline: gpu tests + per-config timings
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python scripts/perf_configs.py grid1001 ico8 torus height batch > gpurun_out/perf_base.json 2>gpurun_out/perf_base.err; cat gpurun_out/perf_base.json | head -c 3000
