# round 2 (session 2), 1 GPU: the L2 Bloom filter now also in front of c2's hash
# (threshold 4 bits per key) -- the 1-GPU suite, c2 K2 ncu --set full (DRAM bytes
# for the bench roofline), the default bench line twice
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02ab_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02ab_tests.log
B2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate"
$B2 > gpurun_out/r02ab_c2_short.json 2> gpurun_out/r02ab_c2_short.err && echo "c2 short ok"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 50 -c 1 -o gpurun_out/r02ab_prof_k2_c2 $B2 > gpurun_out/r02ab_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
ncu -i gpurun_out/r02ab_prof_k2_c2.ncu-rep --page raw --csv > gpurun_out/r02ab_ncu_k2_c2_raw.csv 2>/dev/null; echo "export rc=$?"
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r02ab_bench_$i.json 2> gpurun_out/r02ab_bench_$i.err; echo "bench $i rc=$?"; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ab_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02ab_smoke.log
