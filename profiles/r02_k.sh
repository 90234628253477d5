# round 2 (session 2), 2 GPUs: K2 variants as template instantiations (the
# peer-access branch had cost the plain c2 K2 1.18 -> 1.45 ms); warp-aggregated
# scatter-add (GCP_WAGG=1) parity + timing on c2 / c4; NVML NVLink counter probe;
# the 2-GPU c2 line with NVLink bytes; peer-access two-sided parity again
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "wagg or slot_order or gradient_parity" > gpurun_out/r02k_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02k_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02k_bench_c2.json 2> gpurun_out/r02k_bench_c2.err; echo "c2 rc=$?"
GCP_WAGG=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate > gpurun_out/r02k_bench_c2_wagg.json 2> gpurun_out/r02k_bench_c2_wagg.err; echo "c2 wagg rc=$?"
GCP_WAGG=1 timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02k_bench_c4_wagg.json 2> gpurun_out/r02k_bench_c4_wagg.err; echo "c4 wagg rc=$?"
timeout 300 python tools/nvlink_probe.py 2e9 > gpurun_out/r02k_nvlink_probe.json 2> gpurun_out/r02k_nvlink_probe.err; echo "probe rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 \
    bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02k_c2_n2.json 2> gpurun_out/r02k_c2_n2.err; echo "c2 n2 rc=$?"
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "twosided_peer-2 or sync-2" > gpurun_out/r02k_dist.log 2>&1
echo "dist rc=$?"; tail -3 gpurun_out/r02k_dist.log
