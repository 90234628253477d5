# round 2 last knob, 1 GPU: c3's K2 (d = 5, the non-small geometry) at 2 CTAs/SM
# x one round (default), 3 CTAs/SM x one round (libgcp_n3.so), 2 CTAs/SM x two
# rounds (libgcp_r10.so)
mkdir -p gpurun_out
for v in "" _n3 _r10; do
  GCP_LIB=libgcp$v.so timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02af_c3$v.json 2> gpurun_out/r02af_c3$v.err
  echo "c3 $v rc=$?"; grep -o '"grad": [0-9.]*' gpurun_out/r02af_c3$v.json | head -1
done
