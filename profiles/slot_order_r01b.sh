#!/bin/bash
# slot ordering as a counting sort (3 launches): parity, then c4 at 1 GPU (default = on),
# c4 with it off, c2 (default = off) and c2 forced on
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "slot_order or fit_matches" > gpurun_out/so2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/so2_tests.log
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/so2_c4_on.json 2> gpurun_out/so2_c4_on.err; echo "c4 on rc=$?"
GCP_SLOT_ORDER=0 timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/so2_c4_off.json 2> gpurun_out/so2_c4_off.err; echo "c4 off rc=$?"
GCP_SLOT_ORDER=1 timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/so2_c2_on.json 2> gpurun_out/so2_c2_on.err; echo "c2 on rc=$?"
for f in gpurun_out/so2_c*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],4), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, 'k2', round(d['roofline']['avg_launch_ms'],4), 'launches', d['gpu_launches'])
PY
done
