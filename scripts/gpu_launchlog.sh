#!/bin/bash
# per-launch times of one field for build/ab/<lib>.so: bash scripts/gpu_launchlog.sh "a b" "height torus" [prec]
LIB=paper_1810_08218_b200/libgeodist_b200.so
cp $LIB /tmp/lib_keep.so
for V in $1; do
  cp build/ab/$V.so $LIB
  for w in $2; do echo "== $V $w"; GEODIST_LAUNCH_LOG=1 timeout 120 python scripts/one_field.py $w ${3:-single} 2>&1 | tail -4; done
done
cp /tmp/lib_keep.so $LIB
