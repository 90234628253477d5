# round 2 evidence (1 GPU): (a) c4 K2 / Adam DRAM traffic with the round-2 slot
# order (application replay: --set full's device-memory backup does not fit
# c4); (b) the launch list of the default bench command, filtered to this
# library's kernels (round 1's list was cut off inside torch's generator)
mkdir -p gpurun_out
B4="env GCP_BENCH_ALLOW_SHORT=1 GCP_GRAPHS=0 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B4 > gpurun_out/r02g_c4_short.json 2> gpurun_out/r02g_c4_short.err; echo "c4 bench rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --replay-mode application --metrics $M --clock-control none -k regex:"k_sample|k_adam|k_ord" -s 120 -c 8 --csv --log-file gpurun_out/r02g_ncu_c4_metrics.csv $B4 > gpurun_out/r02g_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
B2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate"
$B2 > gpurun_out/r02g_c2_short.json 2> gpurun_out/r02g_c2_short.err && echo "c2 short ok" && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gcp|k_sample|k_adam|k_reduce|k_init|k_records|k_convert|k_hash|k_dup|k_filter|k_rows" -c 600 --csv --log-file gpurun_out/r02g_launches_c2.csv $B2 > gpurun_out/r02g_ncu_l.log 2>&1
echo "launch list rc=$?"
