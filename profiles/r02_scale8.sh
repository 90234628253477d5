# Staged for an 8-GPU box (gpurun offers this build at most 4): multi-GPU parity
# at P=8 (fused exchange with NVLS multimem, which defaults on from 8 ranks;
# two-sided over NVLink; LocalSGD; FedAdam), then the north-star scaling
# target: c5 (4.69e9 nnz, R=32, p=q=1e8) LocalSGD tau=10 at 8 GPUs against
# its one-GPU 0.225 epochs/s (profiles/r02i_c5_GCP_SLOT_ORDER_0.json; >= 6x
# means >= 1.35 epochs/s), and c2 / c4 sync at 8.
mkdir -p gpurun_out
sed -i 's/@pytest.mark.parametrize("nproc", \[2, 4\])/@pytest.mark.parametrize("nproc", [2, 4, 8])/' tests/test_gpu_dist.py
timeout 1800 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "8" -s > gpurun_out/r02s8_tests.log 2>&1
echo "dist8 rc=$?"; grep -E "DIST-OK|passed|failed" gpurun_out/r02s8_tests.log | tail -8
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29711 bench.py --gpus 8 --config c5 --mode async --tau 10 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02s8_c5_async.json 2> gpurun_out/r02s8_c5_async.err; echo "c5 async rc=$?"
timeout 900 $R --master-port 29712 bench.py --gpus 8 --config c5 --mode sync --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02s8_c5_sync.json 2> gpurun_out/r02s8_c5_sync.err; echo "c5 sync rc=$?"
timeout 600 $R --master-port 29713 bench.py --gpus 8 --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02s8_c4.json 2> gpurun_out/r02s8_c4.err; echo "c4 rc=$?"
timeout 600 $R --master-port 29714 bench.py --gpus 8 --steps 10 --warmup 3 > gpurun_out/r02s8_c2.json 2> gpurun_out/r02s8_c2.err; echo "c2 rc=$?"
