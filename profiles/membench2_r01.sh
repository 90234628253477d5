#!/bin/bash
# membench (incl. contention + shared-memory atomics) and a c3 bench line
mkdir -p gpurun_out
./tools/membench > gpurun_out/membench2.json 2>&1; cat gpurun_out/membench2.json
python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 3000 gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
