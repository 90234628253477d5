#!/bin/bash
# re-run at HEAD (K2 slot order on): DRAM bytes per K2 launch after the change
# c4 (1 GPU): the bench command exits 0 without ncu, then a few single-pass ncu metrics of one
# gradient K2 and one Adam launch (--set full needs a device-memory backup c4 cannot afford)
mkdir -p gpurun_out
B="env GCP_BENCH_ALLOW_SHORT=1 GCP_GRAPHS=0 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/c4h_short.json 2> gpurun_out/c4h_short.err; echo "bench rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:"k_sample|k_adam" -s 60 -c 4 --csv --log-file gpurun_out/ncu_c4h_metrics.csv $B > gpurun_out/ncu_c4h.log 2>&1; echo "ncu rc=$?"
