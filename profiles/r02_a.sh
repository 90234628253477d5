# round 2, first GPU pass: parity suite (new C18 tolerances, slot-order counting
# sort, c4-shaped full-size parity, C17 statistical pin), c4 + c2 bench lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02a_bench_c4.json 2> gpurun_out/r02a_bench_c4.err
echo "c4 rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/r02a_tests.log 2>&1
echo "tests rc=$?"; tail -30 gpurun_out/r02a_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_c2.json 2> gpurun_out/r02a_bench_c2.err
echo "c2 rc=$?"
