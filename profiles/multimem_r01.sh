#!/bin/bash
# NVLS multimem in the fused exchange: dist parity (fp64 + fp32) and c2 / c4 at 4 GPUs, multimem on/off
mkdir -p gpurun_out
[ "${SKIP_TESTS:-0}" = 1 ] || timeout 900 python -m pytest tests/test_gpu_dist.py -q -s -x ${DIST_K:+-k "$DIST_K"} 2>&1 | grep -E "DIST-OK|passed|failed|Error|assert" | head -30
[ "${SKIP_C2:-0}" = 1 ] || for mm in 1 0; do
  GCP_MULTIMEM=$mm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2951$mm bench.py --gpus 4 --no-e2e > gpurun_out/mm${mm}_c2_n4.json 2> gpurun_out/mm${mm}_c2_n4.err
  echo "c2 mm=$mm rc=$?"
done
if [ "${WITH_C4:-0}" = 1 ]; then
for mm in ${C4_MM:-1 0}; do
  GCP_MULTIMEM=$mm timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2952$mm bench.py --gpus 4 --config c4 --no-e2e --steps 3 > gpurun_out/mm${mm}_c4_n4.json 2> gpurun_out/mm${mm}_c4_n4.err
  echo "c4 mm=$mm rc=$?"
done
fi
for f in gpurun_out/mm*_n4.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['value'],3), d['config']['grid'], d['config'].get('exchange'), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()})
    for r in d.get('phase_ms_per_step_ranks') or []: print('   rank', {k: round(v,2) for k,v in r.items()})
except Exception as e:
    print(sys.argv[1], 'unparsed', e)
PY
done
