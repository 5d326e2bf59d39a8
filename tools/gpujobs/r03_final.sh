# round-1 (fifth session) evidence at HEAD: bench lines C1/C3/C4/C5 with the per-family
# roofline notes and 8(d) state model, C2/C3 launch lists, full captures of the C2 generator
# and the C3 NUTS run kernel (summaries only come back)
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r03_smi.txt
for c in c1 c3 c4; do timeout 600 python bench.py --config $c > gpurun_out/r03b_bench_$c.json 2> gpurun_out/r03b_bench_$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03_c2_launches.csv \
  python bench.py --steps 1 --warmup 3 --n 200 --no-cpu --no-lockstep > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03_c3_launches.csv \
  python bench.py --config c3 --steps 1 --warmup 3 --n 100 --no-cpu --no-lockstep > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fsm_run_kernel -s 3 -c 1 \
  -o /tmp/r03_c3run python bench.py --config c3 --steps 1 --warmup 3 --n 100 --no-cpu --no-lockstep > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r03_c3run.ncu-rep > gpurun_out/r03_c3_run.summary.txt 2>&1
python tools/ncu_lines.py /tmp/r03_c3run.ncu-rep 30 > gpurun_out/r03_c3_run.lines.txt 2>&1
ncu -i /tmp/r03_c3run.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/r03_c3_run.dram.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:drmh_draws_kernel -s 20 -c 1 \
  -o /tmp/r03_gen python bench.py --steps 1 --warmup 3 --n 200 --no-cpu --no-lockstep > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r03_gen.ncu-rep > gpurun_out/r03_c2_gen.summary.txt 2>&1
python tools/ncu_lines.py /tmp/r03_gen.ncu-rep 30 > gpurun_out/r03_c2_gen.lines.txt 2>&1
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r03_bench_c5.json 2> gpurun_out/r03_bench_c5.err
