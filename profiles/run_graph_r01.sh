#!/bin/bash
# CUDA-graph epoch replay: GPU suite + c1/c2 bench lines (graphs on and off)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for cfg in c1 c2; do
  python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_${cfg}_graph.json 2> gpurun_out/bench_${cfg}_graph.err
  GCP_GRAPHS=0 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_${cfg}_nograph.json 2> gpurun_out/bench_${cfg}_nograph.err
done
for f in gpurun_out/bench_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('gpu_launches'), d['e2e']['value'])"; done
