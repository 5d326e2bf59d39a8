# HEAD check: GPU suite, smoke, C2 / C2f bench lines with 12 parts
mkdir -p gpurun_out/r05k
export FSMC_HORIZON_OUT=gpurun_out/r05k FSMC_REPORT_OUT=gpurun_out/r05k
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r05k/gpu_suite.log 2>&1; grep -E "passed|failed" gpurun_out/r05k/gpu_suite.log | tail -2
grep -E "bit-exact over" gpurun_out/r05k/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05k/smoke.log 2>&1; tail -1 gpurun_out/r05k/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r05k/bench_c2.json 2> gpurun_out/r05k/bench_c2.err
timeout 900 python bench.py --config c2f --steps 5 --warmup 3 > gpurun_out/r05k/bench_c2f.json 2> gpurun_out/r05k/bench_c2f.err
python tools/bench_table.py gpurun_out/r05k
