#!/bin/bash
# On the GPU box: headline bench line, the ncu launch list of a short bench
# command, fp64/issue counters of the two run kernels, and one --set full
# capture of the step kernel.  Outputs land in gpurun_out/ (summaries -> profiles/).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
echo bench=$?
CMD="python bench.py --steps 2 --warmup 3 --n 200 --no-cpu --no-lockstep"
$CMD > gpurun_out/launch_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/launch_ncu.log 2>&1
echo launches=$?
CMD2="python bench.py --steps 1 --warmup 1 --n 200 --no-cpu --no-lockstep"
$CMD2 > gpurun_out/mix_plain.json 2>&1 && \
  timeout 900 ncu --clock-control none -k regex:"fsm_window_kernel|drmh_draws" -s 20 -c 6 \
    --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
    --csv $CMD2 > gpurun_out/mix_ncu.csv 2> gpurun_out/mix_ncu.err
echo mix=$?
$CMD2 > gpurun_out/full_plain.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsm_window_kernel \
    -s 20 -c 1 -o gpurun_out/prof_c2w $CMD2 > gpurun_out/full_ncu.log 2>&1
echo full=$?
