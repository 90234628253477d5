#!/bin/bash
# per-phase timing of the fused exchange (GCP_FUSED_TRACE=1) at 4 GPUs, c4 and c2, CTA counts 1/2/4 per SM
mkdir -p gpurun_out
for cfg in ${CFGS:-c4 c2}; do
for cps in ${CPS:-1 2 4}; do
  GCP_FUSED_TRACE=1 GCP_FUSED_CTAS_PER_SM=$cps timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$cps bench.py --gpus 4 --config $cfg --no-e2e --steps 1 --warmup 3 > gpurun_out/ftrace_${cfg}_$cps.json 2> gpurun_out/ftrace_${cfg}_$cps.err
  echo "$cfg cps=$cps rc=$?"; grep "fused exchange trace" gpurun_out/ftrace_${cfg}_$cps.err | head -4
done
done
