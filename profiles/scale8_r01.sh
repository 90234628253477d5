# 8 GPUs: dist parity at P=8, then bench at N=8 (c2 sync, fused exchange) and N=8 c2 async
timeout 600 python -m pytest tests/test_gpu_dist.py -q -k "8" 2>&1 | tail -3
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29516 bench.py --gpus 8 --no-e2e > gpurun_out/s8_sync.json 2> gpurun_out/s8_sync.err; echo "sync rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 8 --no-e2e --mode async --tau 10 > gpurun_out/s8_async.json 2> gpurun_out/s8_async.err; echo "async rc=$?"
