#!/bin/bash
# c4 sync and c5 LocalSGD (tau=10) on 2 GPUs
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --config c4 --no-e2e --steps 3 > gpurun_out/c4_n2.json 2> gpurun_out/c4_n2.err; echo "c4 n2 rc=$?"
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 --config c5 --mode async --no-e2e --steps 2 > gpurun_out/c5_n2.json 2> gpurun_out/c5_n2.err; echo "c5 n2 rc=$?"; tail -3 gpurun_out/c5_n2.err
for f in gpurun_out/c4_n2.json gpurun_out/c5_n2.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['value'],4), d['config']['grid'], d['config'].get('exchange'), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()}, d.get('setup_s'))
except Exception as e:
    print(sys.argv[1], 'no line', e)
PY
done
