# round 2: one ncu --set full capture of the c2 gradient K2 at HEAD (the bench
# command exits 0 without ncu first); its DRAM bytes feed the bench roofline
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate"
$B > gpurun_out/r02ncu_c2_plain.json 2> gpurun_out/r02ncu_c2_plain.err && echo "plain ok" && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 50 -c 1 -o gpurun_out/r02_prof_k2_c2 $B > gpurun_out/r02ncu_c2.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r02_prof_k2_c2.ncu-rep --page raw --csv > gpurun_out/r02_ncu_k2_c2_raw.csv 2>/dev/null; echo "export rc=$?"
