# c4 K2: L2 fetch-granularity sweep, then one ncu --set full capture of K2
python tools/k2bench.py --config c4 --iters 10 --l2fetch 0,32,64,128 2>&1 | tail -4
B="python tools/k2bench.py --config c4 --iters 2"
$B > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 6 -c 1 -o gpurun_out/prof_k2_c4 $B > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c4.log
