# round 2: slot order with in-bucket ranks (scatter without reservation atomics),
# conflict-free scan, histogram carried by Adam; parity subset; c4 fuse on/off;
# the full default bench line (c2 + hbm gate c4 + e2e + cpu baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "slot_order or fit_matches or reinit or c4s or lean" > gpurun_out/r02d_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02d_tests.log
for f in 1 0; do
  GCP_ORD_FUSE=$f timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02d_c4_fuse$f.json 2> gpurun_out/r02d_c4_fuse$f.err
  echo "fuse $f rc=$?"
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/r02d_bench.err
