#!/bin/bash
# A/B of build/ab/*.so libraries on named configs + launch log of the current build
# bash scripts/gpu_probe.sh "head pos" "torus height"
LIBS=$1; WHAT=${2:-torus}
mkdir -p gpurun_out
for w in $WHAT; do GEODIST_LAUNCH_LOG=1 timeout 120 python scripts/one_field.py $w single 2>&1 | tail -12; done
[ -n "$LIBS" ] && bash scripts/gpu_ab.sh "$LIBS" "$WHAT"
