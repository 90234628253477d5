# round 2 (session 2), 1 GPU: full-size parity on a c5-shaped tensor (Reddit dims,
# R=32, Poisson, 1e8 nonzeros, p = q = 1e7) in the launch configuration bench.py uses
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k c5s --durations=5 > gpurun_out/r02z_tests.log 2>&1
echo "tests rc=$?"; tail -8 gpurun_out/r02z_tests.log
