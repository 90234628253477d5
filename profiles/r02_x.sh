# round 2 (session 2), 1 GPU: (a) c3 (35 MB of factors: the L2-spill rule turns
# the evict_first policy on) with GCP_L2_HINT=0 / 1; (b) c4 slot-order bucket
# count 2^14 / 2^15 (default) / 2^16 under the final K2 geometry
mkdir -p gpurun_out
for i in 1 2; do for h in 0 1; do
  GCP_L2_HINT=$h timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02x_c3_h${h}_$i.json 2> gpurun_out/r02x_c3_h${h}_$i.err
  echo "c3 h=$h run $i rc=$?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r02x_c3_h${h}_$i.json
done; done
for b in 14 16 15; do
  GCP_ORD_BITS=$b timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02x_c4_bits$b.json 2> gpurun_out/r02x_c4_bits$b.err
  echo "c4 bits=$b rc=$?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r02x_c4_bits$b.json
done
