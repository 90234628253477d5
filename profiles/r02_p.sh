# round 2 (session 2), 4 GPUs: peer-access two-sided with the owed LSA barrier
# after local writes (model init / set / restore) and the owned-rows-only G
# clearing; the whole multi-GPU parity suite (launcher and workers now killed
# as a group on a timeout); the c4 two-sided points again
mkdir -p gpurun_out
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv > gpurun_out/r02p_apps_before.txt 2>&1
timeout 3000 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider --durations=14 > gpurun_out/r02p_dist.log 2>&1
echo "dist rc=$?"; tail -17 gpurun_out/r02p_dist.log
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv > gpurun_out/r02p_apps_after.txt 2>&1; cat gpurun_out/r02p_apps_after.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29750
for s in 1e6 1e7; do
  port=$((port+1))
  timeout 900 $R --master-port $port bench.py --gpus 4 --config c4 --mode twosided --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/r02p_c4_peer_$s.json 2> gpurun_out/r02p_c4_peer_$s.err
  echo "c4 peer $s rc=$?"
done
