# round 2: memory-safety evidence without compute-sanitizer (closed on this
# pool): the bounds-checked build (-DGCP_BOUNDS_CHECK; device indices of the
# hot path checked, violations printed as GCP-BOUNDS) runs tools/sanitize_c1.py
# and the GPU parity suites; the count of GCP-BOUNDS lines must be 0
mkdir -p gpurun_out
export GCP_LIB=libgcp_bounds.so
timeout 900 python tools/sanitize_c1.py > gpurun_out/r02bounds_sanitize.log 2>&1; echo "sanitize_c1 rc=$?"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -s -p no:cacheprovider -k "not c2 and not c3" > gpurun_out/r02bounds_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02bounds_tests.log
echo "GCP-BOUNDS lines: $(cat gpurun_out/r02bounds_sanitize.log gpurun_out/r02bounds_tests.log | grep -c GCP-BOUNDS)"
grep -m5 GCP-BOUNDS gpurun_out/r02bounds_sanitize.log gpurun_out/r02bounds_tests.log
