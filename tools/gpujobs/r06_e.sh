# C1 and C4 DRAM traffic of every launch of a bench run at HEAD (roofline.traffic for their lines)
mkdir -p gpurun_out/r06e
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fsm_run_kernel \
  --csv --log-file gpurun_out/r06e/c1_traffic.csv python bench.py --config c1 --steps 1 --warmup 3 --no-cpu --no-lockstep --no-e2e > gpurun_out/r06e/c1.json 2> gpurun_out/r06e/c1.err
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"fsm_advance|prior_trmm|egress|fsm_run" \
  --csv --log-file gpurun_out/r06e/c4_traffic.csv python bench.py --config c4 --steps 1 --warmup 3 --n 20 --no-cpu --no-lockstep --no-e2e > gpurun_out/r06e/c4.json 2> gpurun_out/r06e/c4.err
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r06e/c1_line.json 2>&1
ls -la gpurun_out/r06e
