# round 2 (session 2), 4 GPUs: the peer-access K2 geometry for remote rows --
# default (3 CTAs/SM x 2 rounds, as the local kernel), 2 CTAs x 4 rounds
# (libgcp_p2r12.so), 4 CTAs x 1 round (libgcp_p4r4.so); c4 two-sided 1e6 / 1e7
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29850
for v in "" _p2r12 _p4r4; do
  for s in 1e6 1e7; do
    port=$((port+1))
    GCP_LIB=libgcp$v.so timeout 900 $R --master-port $port bench.py --gpus 4 --config c4 --mode twosided --samples $s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
        > gpurun_out/r02t_c4_peer${v}_$s.json 2> gpurun_out/r02t_c4_peer${v}_$s.err
    echo "peer $v $s rc=$?"; grep -o '"grad": [0-9.]*' gpurun_out/r02t_c4_peer${v}_$s.json | head -1
  done
done
