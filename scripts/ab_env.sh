#!/bin/bash
# A/B of one build under two environment settings, alternating on one box:
#   bash scripts/ab_env.sh "GEODIST_PERSIST=0" "GEODIST_PERSIST=1" "ico8 torus" [rounds]
EA=$1; EB=$2; WHAT=${3:-ico8}; R=${4:-2}
for r in $(seq $R); do
  for V in A B; do
    if [ $V = A ]; then E=$EA; else E=$EB; fi
    env $E timeout 300 python scripts/perf_configs.py $WHAT 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('$V', ' '.join(f'{k}/{p}={x[\"ms\"]:.3f}' for k,v in d.items() for p,x in v.items()))"
  done
done
