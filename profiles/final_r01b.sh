#!/bin/bash
# re-check at HEAD (after the K2 slot-order change) on 1 B200: GPU suite, smoke(), default bench line,
# the reference arm, and the ncu launch list of the default bench command
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fb_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fb_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/fb_n1.json 2> gpurun_out/fb_n1.err; echo "bench n1 rc=$?"; tail -1 gpurun_out/fb_n1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fb_ref.json 2> gpurun_out/fb_ref.err; echo "ref rc=$?"; tail -1 gpurun_out/fb_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fb_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/fb_ncu.log 2>&1; echo "ncu rc=$?"
