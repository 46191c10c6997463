#!/bin/bash
# One GPU session: tests, smoke, bench (both precisions + reference arm), ncu launch
# list of the bench command, full captures of the solver kernel (ico8 bench workload,
# both precisions; torus wide-band field).  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 300 python bench.py > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err; cut -c1-400 gpurun_out/bench_f32.json
timeout 300 python bench.py --precision double > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err; cut -c1-200 gpurun_out/bench_f64.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-300 gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for P in single double; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:ptp_run4 -s 3 -c 1 -o gpurun_out/prof_${P} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --precision $P > gpurun_out/ncu_${P}.log 2>&1
  tail -1 gpurun_out/ncu_${P}.log
done
# the wide-band launch (MODE 2 instantiation) of the second torus field
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ptp_run4_kernel<float, \(bool\)0, \(int\)2>' -s 1 -c 1 -o gpurun_out/prof_torus_single python scripts/one_torus.py > gpurun_out/ncu_torus.log 2>&1
tail -1 gpurun_out/ncu_torus.log
timeout 600 python scripts/perf_configs.py > gpurun_out/perf_configs.txt 2>&1; tail -3 gpurun_out/perf_configs.txt
timeout 900 python scripts/configs_report.py gpurun_out/configs.json > gpurun_out/configs.log 2>&1; tail -3 gpurun_out/configs.log
