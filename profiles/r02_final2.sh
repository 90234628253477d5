# round 2 final check at the last HEAD (after the 5-way row budget), 1 GPU: the driver's three steps -- pytest -m gpu,
# smoke(), the default bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r02final2_tests.log 2>&1
echo "tests rc=$?"; tail -14 gpurun_out/r02final2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02final2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02final2_smoke.log
timeout 900 python bench.py > gpurun_out/r02final2_bench.json 2> gpurun_out/r02final2_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02final2_ref.json 2> gpurun_out/r02final2_ref.err; echo "ref rc=$?"
