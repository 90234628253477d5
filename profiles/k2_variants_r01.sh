#!/bin/bash
# K2 launch-geometry variants on c2 (one B200): small-row occupancy 4/3/2 CTAs x 256, 8 x 128, 2 x 512
mkdir -p gpurun_out
for lib in libgcp.so libgcp_m3.so libgcp_m2.so libgcp_b128.so libgcp_b512.so libgcp.so; do
  echo "== $lib"; GCP_LIB=$lib timeout 600 python tools/k2bench.py --config ${CFG:-c2} 2>&1 | tail -1
done
