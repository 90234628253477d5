# round 2, 4 GPUs: (a) the 4-GPU parity suite; (b) all-reduce (fused NVLink
# exchange) vs two-sided (device-driven over NVLink windows; and the NCCL
# send/recv variant) against the samples per iteration on c4 (the crossover of
# P:905-923); (c) NVLink data counters (nvidia-smi nvlink -gt d) around one
# fused-exchange run (ncu must not wrap a multi-rank command)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "4" -s > gpurun_out/r02cross4_tests.log 2>&1
echo "dist rc=$?"; grep -E "DIST-OK|passed|failed" gpurun_out/r02cross4_tests.log | tail -8
port=29600
for s in 1e6 1e7 1e8; do
  for m in sync twosided twosided_nccl; do
    port=$((port+1))
    envv=""; mode=$m
    if [ "$m" = "twosided_nccl" ]; then envv="GCP_TWOSIDED_NVL=0"; mode=twosided; fi
    if [ "$m" = "sync" ] && [ "$s" = "1e7" ]; then nvidia-smi nvlink -gt d > gpurun_out/r02cross4_nvlink_before.txt 2>&1; fi
    env $envv timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus 4 --config c4 --mode $mode --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/r02cross4_${m}_$s.json 2> gpurun_out/r02cross4_${m}_$s.err
    echo "$m $s rc=$?"
    if [ "$m" = "sync" ] && [ "$s" = "1e7" ]; then nvidia-smi nvlink -gt d > gpurun_out/r02cross4_nvlink_after.txt 2>&1; fi
  done
done
# c5 at 4 GPUs (LocalSGD tau=10 and sync), for the P=1 -> P=4 ratio
for m in async sync; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29690 \
    bench.py --gpus 4 --config c5 --mode $m --tau 10 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02cross4_c5_$m.json 2> gpurun_out/r02cross4_c5_$m.err
  echo "c5 $m rc=$?"
done
