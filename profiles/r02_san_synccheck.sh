# round 2: compute-sanitizer --tool synccheck over every libgcp kernel on c1-sized
# inputs (tools/sanitize_c1.py); the plain run must exit 0 first
mkdir -p gpurun_out
timeout 600 python tools/sanitize_c1.py > gpurun_out/r02san_plain_synccheck.log 2>&1 && echo "plain ok" && \
timeout 2400 compute-sanitizer --tool synccheck --error-exitcode 3  \
  python tools/sanitize_c1.py > gpurun_out/r02san_synccheck.log 2>&1
echo "synccheck rc=$?"; tail -6 gpurun_out/r02san_synccheck.log
