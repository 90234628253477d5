# round 2 (session 2), 2 GPUs: c5 (Reddit-shaped, 4.69e9 nnz, R=32, p=q=1e8) at
# P = 2 -- each rank's 2.35e9-nonzero block generated into host memory and
# ingested on the lean path; LocalSGD tau=10 and sync, completing c5's 1/2/4 curve
mkdir -p gpurun_out
free -g > gpurun_out/r02y_free.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1800 $R --master-port 29901 bench.py --gpus 2 --config c5 --mode async --tau 10 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02y_c5_async.json 2> gpurun_out/r02y_c5_async.err
echo "c5 async rc=$?"; tail -3 gpurun_out/r02y_c5_async.err
timeout 1800 $R --master-port 29902 bench.py --gpus 2 --config c5 --mode sync --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02y_c5_sync.json 2> gpurun_out/r02y_c5_sync.err
echo "c5 sync rc=$?"; tail -3 gpurun_out/r02y_c5_sync.err
