# headline bench (c2, 1 GPU) + launch list of one timed epoch (gcp kernels only) + ncu --set full of one K2 launch
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
B="python tools/k2bench.py --config c2 --iters 4"
$B > gpurun_out/plain_k2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sample|k_adam|k_reduce" --csv --log-file gpurun_out/launches_k2bench.csv $B > gpurun_out/ncu_l.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 4 -c 1 -o gpurun_out/prof_k2_c2b $B > gpurun_out/ncu_f.log 2>&1
echo "full rc=$?"
