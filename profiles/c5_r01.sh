#!/bin/bash
# c5 (Reddit-shaped, 4.69e9 nnz, R=32, p=q=1e8) on 4 GPUs: per-rank block generation, device ingest;
# LocalSGD tau=10 and sync
mkdir -p gpurun_out
for mode in ${MODES:-async sync}; do
  timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --config c5 --mode $mode --no-e2e --steps 3 --warmup 3 > gpurun_out/c5_${mode}_n4.json 2> gpurun_out/c5_${mode}_n4.err
  echo "c5 $mode rc=$?"; tail -4 gpurun_out/c5_${mode}_n4.err
  python - gpurun_out/c5_${mode}_n4.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],4), d['config']['grid'], d['config'].get('exchange'), d.get('setup_s'), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()}, d['roofline'])
PY
done
