# C2 ncu evidence at HEAD: launch list (bench command, 1 short step), instruction counts per proposal
mkdir -p gpurun_out/r05w
timeout 600 python tools/issue_probe.py 200 > gpurun_out/r05w/plain_probe.json 2>&1 && \
timeout 900 ncu --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__cycles_active.avg,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none \
  -k regex:"drmh_draws|fsm_window" --csv --log-file gpurun_out/r05w/c2_issue.csv python tools/issue_probe.py 200 > gpurun_out/r05w/c2_issue_probe.json 2> gpurun_out/r05w/c2_issue.err
python tools/issue_probe.py --summarise gpurun_out/r05w/c2_issue.csv gpurun_out/r05w/c2_issue_probe.json > gpurun_out/r05w/r05_c2_issue.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r05w/c2_launches.csv \
  python bench.py --steps 1 --warmup 1 --samples 200 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/r05w/c2_launches.csv 4
cat gpurun_out/r05w/r05_c2_issue.json | head -30
