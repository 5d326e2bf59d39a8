# round-1 (third session) final evidence: GPU suite, bench lines C1-C5, reference arm,
# launch lists and full captures of the headline kernels (summaries only come back)
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r02f_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02f_gpu_suite.log 2>&1; tail -1 gpurun_out/r02f_gpu_suite.log
timeout 600 python bench.py > gpurun_out/r02f_bench_c2.json 2> gpurun_out/r02f_bench_c2.err
timeout 300 python bench.py --impl reference > gpurun_out/r02f_bench_c2_reference.json 2>&1
for c in c1 c3 c4; do timeout 900 python bench.py --config $c > gpurun_out/r02f_bench_$c.json 2> gpurun_out/r02f_bench_$c.err; done
timeout 1800 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r02f_bench_c5.json 2> gpurun_out/r02f_bench_c5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_c2_launches.csv \
  python bench.py --steps 1 --warmup 3 --n 200 --no-cpu --no-lockstep > /dev/null 2>&1
for k in drmh_draws_kernel fsm_window_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 \
    -o /tmp/r02f_$k python bench.py --steps 1 --warmup 3 --n 200 --no-cpu --no-lockstep > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/r02f_$k.ncu-rep > gpurun_out/r02f_c2_$k.summary.txt 2>&1
  python tools/ncu_lines.py /tmp/r02f_$k.ncu-rep 30 > gpurun_out/r02f_c2_$k.lines.txt 2>&1
  ncu -i /tmp/r02f_$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/r02f_c2_$k.dram.csv 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:logreg_tc -s 1 -c 1 \
  -o /tmp/r02f_tc python tools/tc_probe.py 18944 bf16-tc 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r02f_tc.ncu-rep > gpurun_out/r02f_c5_tc.summary.txt 2>&1
ncu -i /tmp/r02f_tc.ncu-rep --page raw --csv --metrics sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,gpu__time_duration.sum > gpurun_out/r02f_c5_tc.raw.csv 2>&1
timeout 300 python tools/tc_probe.py 131072 bf16-tc 5 > gpurun_out/r02f_tc_probe.txt 2>&1
