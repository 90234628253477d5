#!/bin/bash
# full GPU suite on 4 GPUs, then c2 / c4 sync at 4 GPUs (fused exchange, unicast, 1 CTA/SM, 4 vectors in flight)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "DIST-OK|passed|failed|Error|assert" | head -30
for cfg in c2 c4; do
  GCP_FUSED_TRACE=${TRACE:-0} timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --config $cfg --no-e2e > gpurun_out/f3_${cfg}_n4.json 2> gpurun_out/f3_${cfg}_n4.err
  echo "$cfg rc=$?"; grep "fused exchange trace" gpurun_out/f3_${cfg}_n4.err | head -1
  python - gpurun_out/f3_${cfg}_n4.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],3), d['config']['grid'], d['config'].get('exchange'), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()})
PY
done
