set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 620 -c 210 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 8 -c 1 -o gpurun_out/prof_k2_c2 $B > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_adam -s 8 -c 1 -o gpurun_out/prof_k3_c2 $B > gpurun_out/ncu_full3.log 2>&1
echo full3 rc=$?
