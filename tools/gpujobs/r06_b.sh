# e2e legs with >= 3 warm-ups and a mean over timed calls; C2 DRAM traffic of every launch at HEAD; full captures of the pair
mkdir -p gpurun_out/r06b
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r06b/bench_c2.json 2> gpurun_out/r06b/bench_c2.err; tail -c 600 gpurun_out/r06b/bench_c2.json
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/r06b/bench_c1.json 2> gpurun_out/r06b/bench_c1.err
timeout 600 python -m pytest tests/test_gpu_bench_multirank.py -q -p no:cacheprovider > gpurun_out/r06b/multirank.log 2>&1; tail -1 gpurun_out/r06b/multirank.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"drmh_draws|fsm_window" \
  --csv --log-file gpurun_out/r06b/c2_traffic.csv python tools/issue_probe.py 200 > gpurun_out/r06b/c2_probe.json 2> gpurun_out/r06b/c2_probe.err
for k in drmh_draws_ilp fsm_window_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 \
    -o /tmp/r06b_$k python tools/issue_probe.py 200 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/r06b_$k.ncu-rep > gpurun_out/r06b/c2_$k.summary.txt 2>&1
  ncu -i /tmp/r06b_$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed.sum > gpurun_out/r06b/c2_$k.dram.csv 2>&1
done
ls gpurun_out/r06b
