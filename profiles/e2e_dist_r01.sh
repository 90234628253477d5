#!/bin/bash
# multi-GPU parity (incl. replace-ingest on one context) and the 2/4-GPU bench lines
# after caching the slice communicators and the symmetric windows across jobs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/e2ed_tests.log 2>&1; echo "dist tests rc=$?"; tail -2 gpurun_out/e2ed_tests.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n > gpurun_out/e2ed_n$n.json 2> gpurun_out/e2ed_n$n.err; echo "bench n$n rc=$?"
done
for f in gpurun_out/e2ed_n2.json gpurun_out/e2ed_n4.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],3), 'e2e', d['e2e']['value'], d['e2e']['phase_ms_rank0'], 'create', d['e2e']['context_create_ms_untimed'])
PY
done
