#!/bin/bash
# ncu --set full of the wide launch (MODE 2) for build/ab/<lib>.so on a field
# bash scripts/gpu_ncu_ab.sh "head pos" "torus height"
LIBS=$1; WHAT=${2:-torus}
LIB=paper_1810_08218_b200/libgeodist_b200.so
cp $LIB /tmp/lib_keep.so
mkdir -p gpurun_out
for V in $LIBS; do
  cp build/ab/$V.so $LIB
  for w in $WHAT; do
    lab=0; [ "$w" = height ] && lab=1
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ptp_run4_kernel<float, \(bool\)$lab, \(int\)2>" -s 1 -c 1 -o gpurun_out/ncu_${V}_${w} python scripts/one_field.py $w > gpurun_out/ncu_${V}_${w}.log 2>&1
    tail -1 gpurun_out/ncu_${V}_${w}.log
  done
done
cp /tmp/lib_keep.so $LIB
