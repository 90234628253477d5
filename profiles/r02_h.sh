# round 2: slot order via fixed-capacity bucket buffers written by the K2
# histogram (no scatter pass); parity subset; c4 bench (fused / standalone)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "slot_order or fit_matches or reinit or c4s or lean" > gpurun_out/r02h_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02h_tests.log
for f in 1 0; do
  GCP_ORD_FUSE=$f timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02h_c4_fuse$f.json 2> gpurun_out/r02h_c4_fuse$f.err
  echo "fuse $f rc=$?"
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate > gpurun_out/r02h_c2.json 2> gpurun_out/r02h_c2.err
echo "c2 rc=$?"
