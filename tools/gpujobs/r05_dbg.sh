# round 2 (session 2), HEAD: compute-sanitizer is closed on this pool, so the whole GPU suite runs
# against a bounds-checked build (variants/debug: FSMC_DEBUG device checks trap on any
# out-of-range index), then the sanitize probe
mkdir -p gpurun_out/r05dbg
FSMC_LIB=$(realpath variants/debug/libfsmc.so) timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r05dbg/debug_suite.log 2>&1; tail -3 gpurun_out/r05dbg/debug_suite.log
FSMC_LIB=$(realpath variants/debug/libfsmc.so) timeout 600 python tools/sanitize_probe.py > gpurun_out/r05dbg/debug_probe.log 2>&1; tail -2 gpurun_out/r05dbg/debug_probe.log
FSMC_LIB=$(realpath variants/debug/libfsmc.so) timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05dbg/debug_bench_c2.json 2>&1; tail -c 300 gpurun_out/r05dbg/debug_bench_c2.json
grep -c "FSMC_CHECK failed" gpurun_out/r05dbg/*.log
