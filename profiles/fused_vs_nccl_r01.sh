# c2 at 4 GPUs: fused NVLink exchange vs NCCL all-reduce exchange, same box
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 4 --no-e2e --steps 10 > gpurun_out/fx_$1.json 2> gpurun_out/fx_$1.err; echo "$1 rc=$?"; }
run fused
GCP_SYNC_EXCHANGE=auto run nccl
run fused2
