# round 2 (session 2) final evidence at HEAD (K2 at 3 CTAs/SM x two row rounds):
# (a) c4 K2 / Adam / ordering DRAM traffic (application replay), (b) ncu --set
# full of the c2 K2, (c) the launch list of the default bench command filtered
# to this library, (d) two default bench lines
mkdir -p gpurun_out
B4="env GCP_BENCH_ALLOW_SHORT=1 GCP_GRAPHS=0 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B4 > gpurun_out/r02u_c4_short.json 2> gpurun_out/r02u_c4_short.err; echo "c4 bench rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --replay-mode application --metrics $M --clock-control none -k regex:"k_sample|k_adam|k_ord" -s 120 -c 8 --csv --log-file gpurun_out/r02u_ncu_c4_metrics.csv $B4 > gpurun_out/r02u_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
B2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate"
$B2 > gpurun_out/r02u_c2_short.json 2> gpurun_out/r02u_c2_short.err && echo "c2 short ok"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 50 -c 1 -o gpurun_out/r02u_prof_k2_c2 $B2 > gpurun_out/r02u_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
ncu -i gpurun_out/r02u_prof_k2_c2.ncu-rep --page raw --csv > gpurun_out/r02u_ncu_k2_c2_raw.csv 2>/dev/null; echo "export rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gcp|k_sample|k_adam|k_reduce|k_init|k_records|k_convert|k_hash|k_dup|k_filter|k_rows" -c 600 --csv --log-file gpurun_out/r02u_launches_c2.csv $B2 > gpurun_out/r02u_ncu_l.log 2>&1
echo "launch list rc=$?"
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r02u_bench_$i.json 2> gpurun_out/r02u_bench_$i.err; echo "bench $i rc=$?"; done
