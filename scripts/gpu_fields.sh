#!/bin/bash
# field-level ncu counters for the bench workloads (scripts/ncu_field.py)
M=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_field; print(ncu_field.METRICS)")
for W in torus1000:torus icosphere8:ico8 grid1001:grid1001; do
  for P in single double; do
    N=${W%%:*}; A=${W##*:}
    timeout 600 ncu --metrics $M --clock-control none -k regex:ptp_run4 --csv --log-file gpurun_out/field_${N}_${P}.csv python scripts/one_field.py $A $P > /dev/null 2>&1
  done
done
ls -la gpurun_out/field_*
