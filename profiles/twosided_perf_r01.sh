#!/bin/bash
# row f3 (two-sided) performance at 4 GPUs on c2 and c4, beside the fused all-reduce layout
mkdir -p gpurun_out
for cfg in c2 c4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --config $cfg --no-e2e --mode twosided --steps 3 > gpurun_out/ts_$cfg.json 2> gpurun_out/ts_$cfg.err
  echo "$cfg twosided rc=$?"; tail -2 gpurun_out/ts_$cfg.err
  python - gpurun_out/ts_$cfg.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],3), d['config']['grid'], d['config'].get('exchange'), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()})
PY
done
