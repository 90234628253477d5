#!/bin/bash
# round-1 final evidence on one B200: GPU tests, the default bench line, then (each only after its
# command exited 0 without ncu) the launch list of the bench command and one ncu --set full K2 capture
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err && echo "short bench ok" && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_l.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 50 -c 1 -o gpurun_out/prof_k2_c2_final $B > gpurun_out/ncu_f.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/prof_k2_c2_final.ncu-rep --page raw --csv > gpurun_out/prof_k2_c2_final_raw.csv 2>/dev/null; echo "export rc=$?"
