# round 2 last: the default bench line at HEAD (c2 roofline skeleton now counts
# the DRAM reads the filter leaves)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02ae_bench.json 2> gpurun_out/r02ae_bench.err; echo "bench rc=$?"
python -c "
import json; b=json.loads(open('gpurun_out/r02ae_bench.json').read().strip().splitlines()[-1]); r=b['roofline']; g=b['hbm_gate']
print(round(b['value'],3), r['bound'], round(r['frac'],3), round(r['avg_launch_ms'],4), b['clocks']['sm_mhz'], b['clocks']['reasons'], '| gate', round(g['epochs_per_s'],3), round(g['frac_of_d4_floor'],3), '| e2e', round(b['e2e']['value'],3))"
