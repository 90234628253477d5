# full GPU suite, c4 at P=4 (fused exchange with unrolled member loads)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 4 --no-e2e --config c4 --steps 5 > gpurun_out/c4p4.json 2> gpurun_out/c4p4.err; echo "c4p4 rc=$?"
