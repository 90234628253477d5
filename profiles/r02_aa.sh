# round 2 (session 2), 1 GPU: the L2 Bloom filter in front of c2's hash under the
# final K2 geometry (5.4 bits per key at the 64-MB cap, GCP_FILTER_MINBITS=4)
# against the plain hash probe (default), twice each
mkdir -p gpurun_out
for i in 1 2; do for m in 12 4; do
  GCP_FILTER_MINBITS=$m timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate > gpurun_out/r02aa_c2_mb${m}_$i.json 2> gpurun_out/r02aa_c2_mb${m}_$i.err
  echo "c2 minbits=$m run $i rc=$?"; grep -o '"grad": [0-9.]*' gpurun_out/r02aa_c2_mb${m}_$i.json | head -1; grep -o '"filter": [a-z]*' gpurun_out/r02aa_c2_mb${m}_$i.json | head -1
done; done
