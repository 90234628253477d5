#!/bin/bash
# slot ordering: counting sort (division-free keys) vs cub radix (16-bit keys) on c4,
# then the launch times of the ordering kernels (ncu launch list, one variant each)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "slot_order or fit_matches" > gpurun_out/so3_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/so3_tests.log
GCP_SLOT_SORT=radix timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "slot_order or fit_matches" > gpurun_out/so3_tests_radix.log 2>&1; echo "tests radix rc=$?"; tail -1 gpurun_out/so3_tests_radix.log
for v in count radix; do
  GCP_SLOT_SORT=$v timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/so3_c4_$v.json 2> gpurun_out/so3_c4_$v.err; echo "c4 $v rc=$?"
done
for f in gpurun_out/so3_c4_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],4), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, 'k2', round(d['roofline']['avg_launch_ms'],4), 'launches', d['gpu_launches'])
PY
done
for v in count radix; do
  GCP_SLOT_SORT=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:slot|Radix|Scan|k_sample' -c 40 --csv --log-file gpurun_out/so3_ncu_$v.csv python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > /dev/null 2>&1; echo "ncu $v rc=$?"
  python - "$v" <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(f"gpurun_out/so3_ncu_{sys.argv[1]}.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki][:60]].append(float(r[vi].replace(',','')))
for k,v in agg.items(): print(sys.argv[1], k, len(v), round(sum(v)/len(v)/1e3,1), "us")
PY
done
