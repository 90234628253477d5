# round 2 (session 2), 1 GPU: L2 evict_first policy on the single-use record /
# hash-bucket reads (GCP_L2_HINT=1) A/B on c2 and c4; NVLink counter probe v2 needs 2 GPUs (separate)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "gradient_parity or membership" > gpurun_out/r02l_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02l_tests.log
for h in 0 1 0 1; do
GCP_L2_HINT=$h timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02l_c2_h$h.json 2> gpurun_out/r02l_c2_h$h.err; echo "c2 h$h rc=$?"
grep -o '"grad": [0-9.]*' gpurun_out/r02l_c2_h$h.json | head -2
done
