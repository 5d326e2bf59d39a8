# round 2 (session 3) final at HEAD: GPU suite, smoke, every bench line, reference arm, C2 launch list
mkdir -p gpurun_out/r06
export FSMC_HORIZON_OUT=gpurun_out/r06 FSMC_REPORT_OUT=gpurun_out/r06
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r06/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r06/gpu_suite.log 2>&1; grep -E "passed|failed" gpurun_out/r06/gpu_suite.log | tail -2
grep -E "bit-exact over|C5 shape|fp32 vs" gpurun_out/r06/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r06/smoke.log 2>&1; tail -1 gpurun_out/r06/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r06/bench_c2.json 2> gpurun_out/r06/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r06/bench_c2_reference.json 2>&1
for c in c1 c3 c4 c2f c3f; do timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r06/bench_$c.json 2> gpurun_out/r06/bench_$c.err; done
timeout 2400 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r06/bench_c5.json 2> gpurun_out/r06/bench_c5.err
python tools/bench_table.py gpurun_out/r06
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r06/c2_launches.csv \
  python bench.py --steps 1 --warmup 1 --samples 200 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/r06/c2_launches.csv 4 > gpurun_out/r06/c2_launch_shares.md
