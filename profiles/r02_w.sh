# round 2 (session 2), 1 GPU: the next iteration's slot-order scan + scatter on
# a side stream concurrent with Adam (GCP_ORD_SIDE=1, default) vs in line
# (GCP_ORD_SIDE=0) on c4, twice each; the 1-GPU parity suite
mkdir -p gpurun_out
for i in 1 2; do for v in 0 1; do
  GCP_ORD_SIDE=$v timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02w_c4_side${v}_$i.json 2> gpurun_out/r02w_c4_side${v}_$i.err
  echo "c4 side=$v run $i rc=$?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r02w_c4_side${v}_$i.json
done; done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02w_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02w_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02w_smoke.log
