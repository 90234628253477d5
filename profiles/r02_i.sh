# round 2: tiled slot order for large p + q (c5 at one GPU: 2e8 slots); parity
# of the tiled order; c5 with 128-MB / 64-MB tiles and with the order off; c4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "slot_order or fit_matches" > gpurun_out/r02i_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02i_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02i_c4.json 2> gpurun_out/r02i_c4.err; echo "c4 rc=$?"
for v in "GCP_ORD_TILE_MB=128" "GCP_ORD_TILE_MB=64" "GCP_SLOT_ORDER=0"; do
  tag=$(echo $v | tr '=' '_')
  env $v timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02i_c5_$tag.json 2> gpurun_out/r02i_c5_$tag.err
  echo "c5 $v rc=$?"
done
