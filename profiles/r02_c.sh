# round 2: slot order with the nonzero lookup table, coalesced scan / scatter and
# the histogram pass fused into Adam; lean ingest parity; c4 bench fused vs not;
# launch list of the c4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "slot_order or fit_matches or reinit or c4s or lean" > gpurun_out/r02c_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02c_tests.log
for f in 1 0; do
  GCP_ORD_FUSE=$f timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02c_c4_fuse$f.json 2> gpurun_out/r02c_c4_fuse$f.err
  echo "fuse $f rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ord|k_sample|k_adam|k_reduce" -s 1500 -c 40 --csv --log-file gpurun_out/r02c_launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02c_ncu.log 2>&1
echo "ncu rc=$?"
