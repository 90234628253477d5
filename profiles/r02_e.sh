# round 2: slot-order histogram carried by K2, scatter carried by Adam (steady
# state: only the scan launches); parity subset; c4 bench; default bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "slot_order or fit_matches or reinit or c4s or lean" > gpurun_out/r02e_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02e_tests.log
for f in 1 0; do
  GCP_ORD_FUSE=$f timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02e_c4_fuse$f.json 2> gpurun_out/r02e_c4_fuse$f.err
  echo "fuse $f rc=$?"
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/r02e_bench.err
