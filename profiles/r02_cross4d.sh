# round 2, 4 GPUs: device-driven two-sided after the pull kernel + k_adam split, import per vector with four in flight (a warp per
# 32-row bitmap word, member words and G rows loaded in parallel): parity at
# 4 GPUs, then the sweep again for the two-sided layout
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "twosided-4 or twosided-2" -s > gpurun_out/r02cross4d_tests.log 2>&1
echo "dist rc=$?"; grep -E "DIST-OK|passed|failed" gpurun_out/r02cross4d_tests.log | tail -8
port=29650
for s in 1e6 1e7 1e8; do
  port=$((port+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port \
    bench.py --gpus 4 --config c4 --mode twosided --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02cross4d_twosided_$s.json 2> gpurun_out/r02cross4d_twosided_$s.err
  echo "twosided $s rc=$?"
done
