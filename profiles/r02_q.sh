# round 2 (session 2), 1 GPU: K2 memory-level parallelism for DRAM-resident
# factors -- small-row geometry (D*NV <= 3: c2, c4) at 4 CTAs/SM with one round
# of row loads in flight (default) vs 2 CTAs/SM with 2 or 4 rounds (m2r8,
# m2r12) and 3 CTAs/SM with 2 rounds (m3r8); c4 and c2
mkdir -p gpurun_out
for v in "" _m2r8 _m2r12 _m3r8; do
  GCP_LIB=libgcp$v.so timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02q_c4$v.json 2> gpurun_out/r02q_c4$v.err
  echo "c4 $v rc=$?"; grep -o '"grad": [0-9.]*' gpurun_out/r02q_c4$v.json | head -1
  GCP_LIB=libgcp$v.so timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-gate > gpurun_out/r02q_c2$v.json 2> gpurun_out/r02q_c2$v.err
  echo "c2 $v rc=$?"; grep -o '"grad": [0-9.]*' gpurun_out/r02q_c2$v.json | head -1
done
