# compute-sanitizer --tool racecheck over every kernel family (tools/sanitize_probe.py); one tool per call
mkdir -p gpurun_out/r04san
timeout 600 python tools/sanitize_probe.py > gpurun_out/r04san/plain_racecheck.log 2>&1 && \
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 python tools/sanitize_probe.py > gpurun_out/r04san/racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r04san/racecheck.log
tail -8 gpurun_out/r04san/racecheck.log
