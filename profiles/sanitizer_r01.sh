# compute-sanitizer memcheck on the smoke path (c1-sized) and the fp64 + u128 parity tests
python __graft_entry__.py smoke > gpurun_out/smoke_plain.log 2>&1 && echo plain-ok && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 3 python __graft_entry__.py smoke > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/memcheck.log
