# K2 tuning variants (tools/k2bench.py on c2); GCP_LIB selects the variant build
for v in libgcp.so libgcp_m3.so libgcp_m4.so libgcp_m2r16.so libgcp_b128m4.so; do
  echo -n "$v "; GCP_LIB=$v python tools/k2bench.py --iters 20 2>&1 | tail -1
done
