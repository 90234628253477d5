#!/bin/bash
# c3 (5-way, u128 keys, Bernoulli) sync at 1, 2, 4 GPUs
mkdir -p gpurun_out
python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/c3_n1.json 2> gpurun_out/c3_n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --config c3 --no-e2e > gpurun_out/c3_n$n.json 2> gpurun_out/c3_n$n.err; echo "n$n rc=$?"
done
for f in gpurun_out/c3_n*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],3), d['config']['grid'], d['config'].get('exchange'), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()})
PY
done
