#!/bin/bash
# GPU test-suite + A/B of library builds: bash scripts/gpu_check.sh "lib_a lib_b" "torus ico8"
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
[ -n "$1" ] && bash scripts/gpu_ab.sh "$1" "${2:-torus}"
