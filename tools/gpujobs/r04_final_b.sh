# round 2 final (b): ncu launch lists and full captures of the headline kernels (C2), the
# C2 instruction counts, C4/C5 launch lists
mkdir -p gpurun_out/r04f_b
# C5 epilogue: log1p on the FMA pipe (two MUFU ops per element) vs the three-MUFU form
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused" > gpurun_out/r04f_b/fused_tests.log 2>&1; tail -1 gpurun_out/r04f_b/fused_tests.log
for L in paper_2503_17405_b200/libfsmc.so variants/sp0/libfsmc.so paper_2503_17405_b200/libfsmc.so; do
  echo $L; FSMC_LIB=$(realpath $L) timeout 300 python tools/tc_probe.py 131072 fp16-tc 3; FSMC_LIB=$(realpath $L) timeout 300 python tools/tc_probe.py 18944 fp16-tc 5
done > gpurun_out/r04f_b/c5_epilogue_ab.txt 2>&1; cat gpurun_out/r04f_b/c5_epilogue_ab.txt
timeout 600 python tools/issue_probe.py 200 > gpurun_out/r04f_b/plain_probe.json 2>&1 && \
timeout 600 ncu --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__cycles_active.avg,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none \
  -k regex:"drmh_draws|fsm_window" --csv --log-file gpurun_out/r04f_b/c2_issue.csv python tools/issue_probe.py 200 > gpurun_out/r04f_b/c2_issue_probe.json 2> gpurun_out/r04f_b/c2_issue.err
python tools/issue_probe.py --summarise gpurun_out/r04f_b/c2_issue.csv gpurun_out/r04f_b/c2_issue_probe.json > gpurun_out/r04f_b/r04_c2_issue.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04f_b/c2_launches.csv \
  python bench.py --steps 1 --warmup 1 --n 200 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
for k in drmh_draws_ilp fsm_window_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 \
    -o /tmp/r04fb_$k python tools/issue_probe.py 200 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/r04fb_$k.ncu-rep > gpurun_out/r04f_b/c2_$k.summary.txt 2>&1
  python tools/ncu_lines.py /tmp/r04fb_$k.ncu-rep 40 > gpurun_out/r04f_b/c2_$k.lines.txt 2>&1
  ncu -i /tmp/r04fb_$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed.sum > gpurun_out/r04f_b/c2_$k.dram.csv 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04f_b/c4_launches.csv \
  python bench.py --config c4 --steps 1 --warmup 1 --n 20 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prior_trmm -s 10 -c 1 \
  -o /tmp/r04fb_trmm python bench.py --config c4 --steps 1 --warmup 1 --n 20 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r04fb_trmm.ncu-rep > gpurun_out/r04f_b/c4_prior_trmm.summary.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:logreg_tc -s 1 -c 1 \
  -o /tmp/r04fb_tc python tools/tc_probe.py 18944 fp16-tc 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r04fb_tc.ncu-rep > gpurun_out/r04f_b/c5_tc.summary.txt 2>&1
ncu -i /tmp/r04fb_tc.ncu-rep --page raw --csv --metrics sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,gpu__time_duration.sum > gpurun_out/r04f_b/c5_tc.raw.csv 2>&1
ls gpurun_out/r04f_b
