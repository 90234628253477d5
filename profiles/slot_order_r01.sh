#!/bin/bash
# slot ordering (GCP_SLOT_ORDER): parity, then c4 and c2 at 1 GPU with it off / on
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "slot_order or fit_matches" > gpurun_out/so_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/so_tests.log
for o in 0 1; do
  GCP_SLOT_ORDER=$o timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/so_c4_$o.json 2> gpurun_out/so_c4_$o.err; echo "c4 order=$o rc=$?"
done
for o in 0 1; do
  GCP_SLOT_ORDER=$o timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/so_c2_$o.json 2> gpurun_out/so_c2_$o.err; echo "c2 order=$o rc=$?"
done
for f in gpurun_out/so_c*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],4), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, 'k2', round(d['roofline']['avg_launch_ms'],4), 'launches', d['gpu_launches'])
PY
done
