#!/bin/bash
# K2 with the shared-memory staged lookahead (cp.async, GCP_SMEM_STAGES = 2/3/4/6) vs the register pipeline
mkdir -p gpurun_out
GCP_LIB=libgcp_s3.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for lib in libgcp.so libgcp_s2.so libgcp_s3.so libgcp_s4.so libgcp_s6.so libgcp.so; do
  for cfg in ${CFGS:-c2 c4}; do
    echo "== $lib $cfg"; GCP_LIB=$lib timeout 600 python tools/k2bench.py --config $cfg --iters 10 2>&1 | tail -1 | grep -o '"grad_ms": [0-9.]*\|"loss_ms": [0-9.]*' | tr '\n' ' '; echo
  done
done
