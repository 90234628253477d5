# round 2 (session 2), 2 GPUs: warp-aggregated scatter fixed (the shuffles now
# read an unmodified copy) -- parity + timing again; two-sided parity with peer
# access as the default and the import/export kernels forced; then the
# single-GPU evidence of profiles/r02_n.sh (ncu captures, launch list, bench lines)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "warp_aggregated or slot_order or gradient_parity" > gpurun_out/r02o_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02o_tests.log
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "twosided" > gpurun_out/r02o_dist.log 2>&1
echo "dist rc=$?"; tail -3 gpurun_out/r02o_dist.log
GCP_WAGG=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02o_bench_c2_wagg.json 2> gpurun_out/r02o_bench_c2_wagg.err; echo "c2 wagg rc=$?"
grep -o '"grad": [0-9.]*' gpurun_out/r02o_bench_c2_wagg.json | head -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 \
    bench.py --gpus 2 --config c4 --mode twosided --samples 1e6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02o_c4_ts_1e6.json 2> gpurun_out/r02o_c4_ts_1e6.err; echo "c4 ts rc=$?"
bash profiles/r02_n.sh
