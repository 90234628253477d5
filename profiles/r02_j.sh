# round 2 (session 2), 2 GPUs: HEAD re-check after the container re-creation --
# full GPU suite (1- and 2-GPU cases, incl. two-sided by peer access), smoke,
# default bench line, then the peer-access two-sided c4 points at 2 GPUs
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02j_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r02j_tests.log 2>&1
echo "tests rc=$?"; tail -14 gpurun_out/r02j_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02j_smoke.log
timeout 900 python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc=$?"
for s in 1e6 1e7; do
  for v in peer 1; do
  GCP_TWOSIDED_NVL=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2966${s:2:1} \
    bench.py --gpus 2 --config c4 --mode twosided --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02j_ts_${v}_$s.json 2> gpurun_out/r02j_ts_${v}_$s.err
  echo "twosided $v $s rc=$?"
  done
done
