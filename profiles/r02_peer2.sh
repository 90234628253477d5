# round 2, 2 GPUs: two-sided by peer access (K2 gathers owners' rows and
# red.adds into owners' G over NVLink): parity, then c4 at 1e6 / 1e7 samples
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "twosided_peer-2" -s > gpurun_out/r02peer2_tests.log 2>&1
echo "dist rc=$?"; grep -E "DIST-OK|passed|failed|Error|error" gpurun_out/r02peer2_tests.log | tail -8
for s in 1e6 1e7; do
  GCP_TWOSIDED_NVL=peer timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2966${s:2:1} \
    bench.py --gpus 2 --config c4 --mode twosided --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02peer2_$s.json 2> gpurun_out/r02peer2_$s.err
  echo "peer $s rc=$?"
done
