timeout 600 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_c2_ref.json 2>&1
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c2_launches.csv \
  python bench.py --steps 1 --warmup 3 --n 200 --no-cpu --no-lockstep > /dev/null 2>&1
