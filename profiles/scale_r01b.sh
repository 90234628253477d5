# multi-GPU with the fused NVLink exchange: parity at P=2,4, bench at N=1,2,4 (c2, sync)
timeout 600 python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -3
for n in 1 2 4; do
  if [ $n = 1 ]; then timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/scaleb_n1.json 2> gpurun_out/scaleb_n1.err
  else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $n --no-e2e > gpurun_out/scaleb_n$n.json 2> gpurun_out/scaleb_n$n.err; fi
  echo "N=$n rc=$?"
done
