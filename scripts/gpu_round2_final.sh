#!/bin/bash
# Round-2 evidence pass (one GPU): GPU tests + smoke, bench lines (both arms), the ncu
# launch list of the bench command, field-level ncu counters for the bench workloads,
# full ncu captures of the dominant launches.  Outputs in gpurun_out/r2/.
set -u
O=gpurun_out/r2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1300 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_torus_f32.json 2> $O/bench_torus_f32.err; cut -c1-300 $O/bench_torus_f32.json
timeout 600 python bench.py --precision double > $O/bench_torus_f64.json 2> $O/bench_torus_f64.err; cut -c1-200 $O/bench_torus_f64.json
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; cut -c1-300 $O/bench_reference.json
for W in icosphere8 grid1001; do
  timeout 600 python bench.py --workload $W > $O/bench_${W}_f32.json 2> $O/bench_${W}.err; cut -c1-200 $O/bench_${W}_f32.json
done
timeout 900 python bench.py --workload batch512 --steps 1 > $O/bench_batch512.json 2> $O/bench_batch512.err; cut -c1-200 $O/bench_batch512.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_torus_f32.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
M=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_field; print(ncu_field.METRICS)")
for W in torus1000:torus icosphere8:ico8 grid1001:grid1001; do
  for P in single double; do
    N=${W%%:*}; A=${W##*:}
    timeout 600 ncu --metrics $M --clock-control none -k regex:ptp_run4 --csv --log-file $O/field_${N}_${P}.csv python scripts/one_field.py $A $P > /dev/null 2>&1
  done
done
# full captures: torus wide launch (fp32, fp64), icosphere-8 narrow launch (fp32)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ptp_run4_kernel<float, \(bool\)0, \(int\)2>' -s 1 -c 1 -o $O/full_torus_wide_f32 python scripts/one_field.py torus single > $O/full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ptp_run4_kernel<double, \(bool\)0, \(int\)2>' -s 1 -c 1 -o $O/full_torus_wide_f64 python scripts/one_field.py torus double > $O/full2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ptp_run4_kernel<float, \(bool\)0, \(int\)1>' -s 1 -c 1 -o $O/full_ico8_f32 python scripts/one_field.py ico8 single > $O/full3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ptp_run4_kernel<float, \(bool\)1, \(int\)2>' -s 1 -c 1 -o $O/full_height_wide_f32 python scripts/one_field.py height single > $O/full4.log 2>&1
ls -la $O | tail -30
