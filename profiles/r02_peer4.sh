# round 2, 4 GPUs: two-sided by peer access -- parity at 2 and 4, the c4 sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "twosided_peer" -s > gpurun_out/r02peer4_tests.log 2>&1
echo "dist rc=$?"; grep -E "DIST-OK|passed|failed|AssertionError" gpurun_out/r02peer4_tests.log | tail -8
for s in 1e6 1e7 1e8; do
  GCP_TWOSIDED_NVL=peer timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2967${s:2:1} \
    bench.py --gpus 4 --config c4 --mode twosided --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02peer4_$s.json 2> gpurun_out/r02peer4_$s.err
  echo "peer $s rc=$?"
done
