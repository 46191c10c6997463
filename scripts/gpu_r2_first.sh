#!/bin/bash
# round-2 first GPU pass: L2 peak, bench lines on the new workloads, GPU test-suite
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/l2_peak.cu -o /tmp/l2_peak && /tmp/l2_peak > gpurun_out/l2_peak.json
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv >> gpurun_out/l2_peak.json
python bench.py --steps 5 --warmup 3 > gpurun_out/b_torus.json 2> gpurun_out/b_torus.err
python bench.py --workload icosphere8 --steps 5 --no-cpu-baseline > gpurun_out/b_ico.json 2>&1
python bench.py --workload grid1001 --steps 5 --no-cpu-baseline > gpurun_out/b_grid.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
