# round 2 (session 2), 4 GPUs: c2 at 2 and 4 GPUs with the L2 Bloom filter now
# in front of each rank's hash (default flags, e2e included)
mkdir -p gpurun_out
port=29950
for n in 2 4; do
  port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r02ac_c2_n$n.json 2> gpurun_out/r02ac_c2_n$n.err
  echo "c2 n$n rc=$?"; grep -o '"value": [0-9.]*' gpurun_out/r02ac_c2_n$n.json | head -2
done
