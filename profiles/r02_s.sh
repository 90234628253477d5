# round 2 (session 2), 4 GPUs, final: the multi-GPU parity suite at HEAD; c2 at
# 2 and 4 GPUs (default flags, e2e included); c4 all-reduce vs two-sided (peer
# access) at 1e6 / 1e7 samples with the 3-CTA K2 geometry; c5 LocalSGD tau=10
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/r02s_dist.log 2>&1
echo "dist rc=$?"; tail -3 gpurun_out/r02s_dist.log
port=29800
for n in 2 4; do
  port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r02s_c2_n$n.json 2> gpurun_out/r02s_c2_n$n.err
  echo "c2 n$n rc=$?"
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for s in 1e6 1e7; do
  for m in sync twosided; do
    port=$((port+1))
    timeout 900 $R --master-port $port bench.py --gpus 4 --config c4 --mode $m --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
        > gpurun_out/r02s_c4_${m}_$s.json 2> gpurun_out/r02s_c4_${m}_$s.err
    echo "c4 $m $s rc=$?"
  done
done
port=$((port+1))
timeout 1500 $R --master-port $port bench.py --gpus 4 --config c5 --mode async --tau 10 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02s_c5_async.json 2> gpurun_out/r02s_c5_async.err
echo "c5 async rc=$?"
