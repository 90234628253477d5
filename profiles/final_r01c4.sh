#!/bin/bash
# re-check at HEAD on 4 B200s: the GPU suite (multi-GPU tests included) and the 2/4-GPU bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f4_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f4_tests.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2973$n bench.py --gpus $n > gpurun_out/f4_n$n.json 2> gpurun_out/f4_n$n.err; echo "bench n$n rc=$?"; tail -1 gpurun_out/f4_n$n.json | cut -c1-300
done
