#!/bin/bash
# end-of-round-1 check on 4 B200s: full GPU suite, smoke(), the default bench line (N=1), the
# reference arm (oracle) and the 2/4-GPU bench lines
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo "bench n1 rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n > gpurun_out/final_n$n.json 2> gpurun_out/final_n$n.err; echo "bench n$n rc=$?"
done
for f in gpurun_out/final_n1.json gpurun_out/final_n2.json gpurun_out/final_n4.json gpurun_out/final_ref.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d.get('impl','ours'), round(d['value'],5), d['unit'], 'e2e', (d.get('e2e') or {}).get('value'), 'roofline', (d.get('roofline') or {}).get('frac'), 'clocks', (d.get('clocks') or {}).get('sm_mhz'))
PY
done
