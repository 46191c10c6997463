#!/bin/bash
# A/B of library builds in build/ab/*.so on the torus (+ ncu of the wide launch of the
# current build): bash scripts/gpu_ab.sh "lib_r1 lib_eager lib_lazy" torus [ncu]
LIBS=$1; WHAT=${2:-torus}
LIB=paper_1810_08218_b200/libgeodist_b200.so
cp $LIB /tmp/lib_keep.so
for r in 1 2; do
  for V in $LIBS; do
    cp build/ab/$V.so $LIB
    timeout 300 python scripts/perf_configs.py $WHAT 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('$V', ' '.join(f'{k}/{p}={x[\"ms\"]:.3f}' for k,v in d.items() if isinstance(v, dict) for p,x in v.items()))"
  done
done
cp /tmp/lib_keep.so $LIB
if [ -n "$3" ]; then
  for V in $3; do
    cp build/ab/$V.so $LIB
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ptp_run4_kernel<float, \(bool\)0, \(int\)2>' -s 1 -c 1 -o gpurun_out/prof_wide_$V python scripts/one_field.py torus > gpurun_out/ncu_$V.log 2>&1
    tail -1 gpurun_out/ncu_$V.log
  done
  cp /tmp/lib_keep.so $LIB
fi
