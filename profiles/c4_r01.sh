# c4 (Amazon-shaped, 1.74e9 nnz, R=16, Gaussian) on one B200: the HBM-bound case
timeout 1200 python -X faulthandler bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "c4 rc=$?"; grep -v "^  File\|^    " gpurun_out/bench_c4.err | tail -8; grep -A12 "Fatal Python" gpurun_out/bench_c4.err | head -30; tail -1 gpurun_out/bench_c4.json | cut -c1-2500
