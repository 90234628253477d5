# row f3 (two-sided) parity at P=2,4 and c2 bench at 4 GPUs, vs the all-reduce layout
timeout 900 python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -3
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 4 --no-e2e --mode twosided --steps 5 > gpurun_out/ts4.json 2> gpurun_out/ts4.err; echo "ts4 rc=$?"
