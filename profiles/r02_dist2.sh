# round 2, 2 GPUs: multi-GPU parity (sync fused, sync fp32 + NVLS + slot order,
# two-sided over NVLink windows, two-sided over NCCL, LocalSGD + slot order, FedAdam)
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r02dist2_topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "2" -s > gpurun_out/r02dist2_tests.log 2>&1
echo "dist rc=$?"; grep -E "DIST-OK|passed|failed|Error" gpurun_out/r02dist2_tests.log | tail -15
