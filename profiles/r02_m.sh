# round 2 (session 2), 4 GPUs: the full GPU suite at HEAD (1-, 2- and 4-GPU
# cases), NVML NVLink counter probe, c2 sync at 4 GPUs with the NVLink byte
# counters, c4 at 4 GPUs: sync vs two-sided (NVLink import/export, and by peer
# access) against samples per iteration
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/r02m_tests.log 2>&1
echo "tests rc=$?"; tail -16 gpurun_out/r02m_tests.log
timeout 300 python tools/nvlink_probe.py 2e9 > gpurun_out/r02m_nvlink_probe.json 2> gpurun_out/r02m_nvlink_probe.err; echo "probe rc=$?"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29691 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02m_c2_n4.json 2> gpurun_out/r02m_c2_n4.err; echo "c2 n4 rc=$?"
port=29692
for s in 1e6 1e7 1e8; do
  for v in sync peer nvl; do
    if [ $v = sync ]; then M="--mode sync"; E=""; else M="--mode twosided"; E="GCP_TWOSIDED_NVL=$([ $v = peer ] && echo peer || echo 1)"; fi
    port=$((port+1))
    env $E timeout 900 $R --master-port $port bench.py --gpus 4 --config c4 $M --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/r02m_c4_${v}_$s.json 2> gpurun_out/r02m_c4_${v}_$s.err
    echo "c4 $v $s rc=$?"
  done
done
