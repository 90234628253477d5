#!/bin/bash
# fused exchange grid size (adaptive vs full 148) at 4 GPUs on c2, with phase traces
mkdir -p gpurun_out
for gr in ${GRIDS:-0 148 16 32 64}; do
  GCP_FUSED_GRID=$gr GCP_FUSED_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2958$((gr % 10)) bench.py --gpus 4 --no-e2e --steps 3 > gpurun_out/fg_$gr.json 2> gpurun_out/fg_$gr.err
  echo "grid=$gr rc=$?"; grep "fused exchange trace" gpurun_out/fg_$gr.err | head -1
  GCP_FUSED_GRID=$gr timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2959$((gr % 10)) bench.py --gpus 4 --no-e2e > gpurun_out/fgv_$gr.json 2> gpurun_out/fgv_$gr.err
  python - gpurun_out/fgv_$gr.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],3), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()})
PY
done
