# C3 DRAM traffic of every fsm_run_kernel launch at HEAD (shared-memory trajectory ends, compile-time state visits); one full capture
mkdir -p gpurun_out/r06d
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fsm_run_kernel \
  --csv --log-file gpurun_out/r06d/c3_traffic.csv python bench.py --config c3 --steps 1 --warmup 3 --n 100 --no-cpu --no-lockstep --no-e2e > gpurun_out/r06d/c3_probe.json 2> gpurun_out/r06d/c3_probe.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fsm_run_kernel -s 3 -c 1 \
  -o /tmp/r06d_c3run python bench.py --config c3 --steps 1 --warmup 3 --n 100 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r06d_c3run.ncu-rep > gpurun_out/r06d/c3_run.summary.txt 2>&1
python tools/ncu_lines.py /tmp/r06d_c3run.ncu-rep 30 > gpurun_out/r06d/c3_run.lines.txt 2>&1
ncu -i /tmp/r06d_c3run.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/r06d/c3_run.dram.csv 2>&1
ls -la gpurun_out/r06d
