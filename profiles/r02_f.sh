# round 2: slot order = histogram in K2 + standalone scan + scatter (default),
# vs scatter in Adam (GCP_ORD_FUSE=2) and everything standalone (0); launch list
mkdir -p gpurun_out
for f in 1 2 0; do
  GCP_ORD_FUSE=$f timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02f_c4_fuse$f.json 2> gpurun_out/r02f_c4_fuse$f.err
  echo "fuse $f rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ord|k_sample|k_adam|k_reduce" -s 1500 -c 40 --csv --log-file gpurun_out/r02f_launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu.log 2>&1
echo "ncu rc=$?"
