# round 2 (session 2), 1 GPU: the small-row K2 geometry at 3 CTAs/SM x two
# rounds of row loads in flight (fp32) as the default -- the 1-GPU parity suite,
# the default bench line, and c5 against the previous geometry (libgcp_m4r4.so)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/r02r_tests.log 2>&1
echo "tests rc=$?"; tail -12 gpurun_out/r02r_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02r_smoke.log
timeout 900 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo "bench rc=$?"
for v in "" _m4r4; do
  GCP_LIB=libgcp$v.so timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02r_c5$v.json 2> gpurun_out/r02r_c5$v.err
  echo "c5 $v rc=$?"; grep -o '"grad": [0-9.]*' gpurun_out/r02r_c5$v.json | head -1
done
