#!/bin/bash
# membench (incl. c4-shaped skeleton), smoke(), c1/c4 1-GPU and c2 sync at N=1,2,4 with the current build
mkdir -p gpurun_out
./tools/membench > gpurun_out/membench3.json 2>&1; tail -c 400 gpurun_out/membench3.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py --config c1 --no-cpu-baseline > gpurun_out/fs_c1.json 2> gpurun_out/fs_c1.err; echo "c1 rc=$?"
python bench.py --config c4 --no-cpu-baseline --steps 3 > gpurun_out/fs_c4.json 2> gpurun_out/fs_c4.err; echo "c4 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n > gpurun_out/fs_c2_n$n.json 2> gpurun_out/fs_c2_n$n.err; echo "c2 n=$n rc=$?"
done
for f in gpurun_out/fs_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],3), d['config'].get('exchange'), 'e2e', round(d['e2e']['value'],3) if d.get('e2e') else None, {k: round(v,2) for k,v in d['phase_ms_per_step'].items()}, d['roofline']['frac'])
PY
done
