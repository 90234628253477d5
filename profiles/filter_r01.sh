#!/bin/bash
# K2 A/B on c2: previous pipeline (libgcp_old) vs two-deep pipeline with / without the L2 Bloom
# filter, small-geometry occupancy 4/3/2 CTAs per SM (libgcp_m3 / libgcp_m2)
mkdir -p gpurun_out
CFG=${CFG:-c2}
run() { echo "== $1 filter=$2 $3"; GCP_LIB=$1 GCP_FILTER=$2 GCP_FILTER_MB=${3:-64} timeout 600 python tools/k2bench.py --config $CFG --strategies ${STRATS:-stratified} 2>&1 | tail -${NS:-1}; }
run libgcp_old.so 1
run libgcp.so 0
run libgcp.so 1
run libgcp_m3.so 1
run libgcp_m2.so 1
run libgcp_m3.so 1 32
run libgcp_m3.so 1 16
