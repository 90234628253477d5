# c2 at 4 GPUs (sync): NCCL protocol variants / exchange policy for the per-iteration exchange
run() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --no-e2e --steps 5 > gpurun_out/nccl_$1.json 2> gpurun_out/nccl_$1.err; echo "$1 rc=$?"; }
run default
NCCL_PROTO=LL run ll
NCCL_PROTO=LL128 run ll128
GCP_SYNC_EXCHANGE=rs run rsag
NCCL_NVLS_ENABLE=0 run nonvls
