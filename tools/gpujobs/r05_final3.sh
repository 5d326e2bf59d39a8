# round 2 (session 2) final at HEAD, third pass (progress check every round): GPU suite, smoke, every bench line, reference arm
mkdir -p gpurun_out/r05h
export FSMC_HORIZON_OUT=gpurun_out/r05h FSMC_REPORT_OUT=gpurun_out/r05h
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r05h/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r05h/gpu_suite.log 2>&1; grep -E "passed|failed" gpurun_out/r05h/gpu_suite.log | tail -2
grep -E "bit-exact over|C5 shape|fp32 vs" gpurun_out/r05h/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05h/smoke.log 2>&1; tail -1 gpurun_out/r05h/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r05h/bench_c2.json 2> gpurun_out/r05h/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r05h/bench_c2_reference.json 2>&1
for c in c1 c3 c4 c2f c3f; do timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r05h/bench_$c.json 2> gpurun_out/r05h/bench_$c.err; done
timeout 2400 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r05h/bench_c5.json 2> gpurun_out/r05h/bench_c5.err
python tools/bench_table.py gpurun_out/r05h
