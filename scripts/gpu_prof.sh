#!/bin/bash
# ncu --set full of one wide (MODE 2) launch: bash scripts/gpu_prof.sh tag "torus|height" [precision] [labels 0|1]
TAG=$1; W=${2:-torus}; P=${3:-single}; L=${4:-0}
T=float; [ "$P" = double ] && T=double
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ptp_run4_kernel<$T, \(bool\)$L, \(int\)2>" -s 1 -c 1 -o gpurun_out/prof_${TAG} python scripts/one_field.py $W $P > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
