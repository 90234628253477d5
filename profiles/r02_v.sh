# round 2 (session 2), 4 GPUs: the multi-GPU parity suite with the rejected-epoch
# fit (restore under every sync-family layout, incl. peer access); then the
# bounds-checked build (-DGCP_BOUNDS_CHECK, libgcp_bounds.so) over every kernel
# on c1-sized inputs, the 1-GPU parity suites, and the 2-GPU sync / two-sided
# cases (peer-access gathers and scatter-adds checked on the device)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/r02v_dist.log 2>&1
echo "dist rc=$?"; tail -3 gpurun_out/r02v_dist.log
export GCP_LIB=libgcp_bounds.so
timeout 900 python tools/sanitize_c1.py > gpurun_out/r02v_bounds_sanitize.log 2>&1; echo "sanitize_c1 rc=$?"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -s -p no:cacheprovider -k "not c2 and not c3" > gpurun_out/r02v_bounds_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02v_bounds_tests.log
timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -q -s -p no:cacheprovider -k "sync-2 or twosided-2 or twosided_peer-2" > gpurun_out/r02v_bounds_dist.log 2>&1; echo "bounds dist rc=$?"
tail -2 gpurun_out/r02v_bounds_dist.log
echo "GCP-BOUNDS lines: $(cat gpurun_out/r02v_bounds_sanitize.log gpurun_out/r02v_bounds_tests.log gpurun_out/r02v_bounds_dist.log | grep -c GCP-BOUNDS)"
grep -m5 GCP-BOUNDS gpurun_out/r02v_bounds_*.log
