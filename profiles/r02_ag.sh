# round 2 last, 1 GPU: two rounds of row loads for 5-way rows (GCP_RBREG 10) --
# the parity suite (incl. the 5-way / u128 cases and full-size c3), c3 bench twice
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "not c2 and not c4s and not c5s" > gpurun_out/r02ag_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02ag_tests.log
for i in 1 2; do
  timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02ag_c3_$i.json 2> gpurun_out/r02ag_c3_$i.err
  echo "c3 $i rc=$?"; grep -o '"grad": [0-9.]*' gpurun_out/r02ag_c3_$i.json | head -1; grep -o '"value": [0-9.]*' gpurun_out/r02ag_c3_$i.json | head -1
done
