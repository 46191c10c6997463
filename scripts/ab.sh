#!/bin/bash
# A/B timing of two builds of the library on the same box, alternating:
#   bash scripts/ab.sh build/libA.so build/libB.so "ico8 torus" [rounds]
A=$1; B=$2; WHAT=${3:-ico8}; R=${4:-3}
LIB=paper_1810_08218_b200/libgeodist_b200.so
cp $LIB /tmp/lib_keep.so
for r in $(seq $R); do
  for V in A B; do
    if [ $V = A ]; then cp $A $LIB; else cp $B $LIB; fi
    timeout 300 python scripts/perf_configs.py $WHAT 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('$V', ' '.join(f'{k}/{p}={x[\"ms\"]:.3f}' for k,v in d.items() for p,x in v.items()))"
  done
done
cp /tmp/lib_keep.so $LIB
