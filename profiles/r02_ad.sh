# round 2 final, 4 GPUs: the whole GPU suite at HEAD (1-, 2- and 4-GPU cases in
# one run), then c3 (5-way LBNL-shaped) at 1 / 2 / 4 GPUs
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=6 > gpurun_out/r02ad_tests.log 2>&1
echo "tests rc=$?"; tail -10 gpurun_out/r02ad_tests.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02ad_c3_n1.json 2> gpurun_out/r02ad_c3_n1.err; echo "c3 n1 rc=$?"
port=29970
for n in 2 4; do
  port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus $n --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02ad_c3_n$n.json 2> gpurun_out/r02ad_c3_n$n.err
  echo "c3 n$n rc=$?"
done
for n in 1 2 4; do grep -o '"value": [0-9.]*' gpurun_out/r02ad_c3_n$n.json | head -1; done
