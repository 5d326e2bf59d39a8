# round 2 final (second pass, at HEAD): GPU suite, smoke, every bench line, reference arm,
# C2 launch list + instruction counts at HEAD, bounds-checked build over the suite
mkdir -p gpurun_out/r04g2
export FSMC_HORIZON_OUT=gpurun_out/r04g2 FSMC_REPORT_OUT=gpurun_out/r04g2
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r04g2/gpu_suite.log 2>&1; grep -E "passed|failed" gpurun_out/r04g2/gpu_suite.log | tail -2
grep -E "bit-exact over|C5 shape|fp32 vs" gpurun_out/r04g2/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04g2/smoke.log 2>&1; tail -1 gpurun_out/r04g2/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r04g2/bench_c2.json 2> gpurun_out/r04g2/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r04g2/bench_c2_reference.json 2>&1
for c in c1 c3 c4 c2f c3f; do timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r04g2/bench_$c.json 2> gpurun_out/r04g2/bench_$c.err; done
timeout 2400 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r04g2/bench_c5.json 2> gpurun_out/r04g2/bench_c5.err
python tools/bench_table.py gpurun_out/r04g2
timeout 600 python tools/issue_probe.py 200 > gpurun_out/r04g2/plain_probe.json 2>&1 && \
timeout 600 ncu --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__cycles_active.avg,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none \
  -k regex:"drmh_draws|fsm_window" --csv --log-file gpurun_out/r04g2/c2_issue.csv python tools/issue_probe.py 200 > gpurun_out/r04g2/c2_issue_probe.json 2> gpurun_out/r04g2/c2_issue.err
python tools/issue_probe.py --summarise gpurun_out/r04g2/c2_issue.csv gpurun_out/r04g2/c2_issue_probe.json > gpurun_out/r04g2/r04_c2_issue.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04g2/c2_launches.csv \
  python bench.py --steps 1 --warmup 1 --samples 200 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/r04g2/c2_launches.csv 4
