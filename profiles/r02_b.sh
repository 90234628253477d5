# round 2: slot-order bucket granularity on c4 (GCP_ORD_BITS 12/14/15), parity of
# the new ordering, and the launch list of the c4 bench (per-kernel device times)
mkdir -p gpurun_out
free -g > gpurun_out/r02b_host.txt; nproc >> gpurun_out/r02b_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r02b_host.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "slot_order or fit_matches or reinit or c4s" > gpurun_out/r02b_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02b_tests.log
for b in 12 14 15; do
  GCP_ORD_BITS=$b timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate > gpurun_out/r02b_c4_bits$b.json 2> gpurun_out/r02b_c4_bits$b.err
  echo "bits $b rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ord|k_sample|k_adam|k_reduce" -s 1500 -c 40 --csv --log-file gpurun_out/r02b_launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate > gpurun_out/r02b_ncu.log 2>&1
echo "ncu rc=$?"
