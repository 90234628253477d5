# round 2: c5 (Reddit-shaped, 4.69e9 nnz, R=32, Poisson, p=q=1e8) on ONE B200:
# generated on the device partition by partition into host memory, lean
# (key, value) ingest, hash set at load <= 0.75; the P=1 baseline of the
# north-star 8-GPU scaling target
mkdir -p gpurun_out
free -g > gpurun_out/r02c5_mem_before.txt
( while true; do nvidia-smi --query-gpu=memory.used,clocks.sm --format=csv,noheader >> gpurun_out/r02c5_gpumem.txt; free -g | grep Mem >> gpurun_out/r02c5_hostmem.txt; sleep 5; done ) &
MON=$!
GCP_INGEST_TRACE=1 timeout 1800 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02c5_bench.json 2> gpurun_out/r02c5_bench.err
echo "c5 rc=$?"
kill $MON
tail -20 gpurun_out/r02c5_bench.err
