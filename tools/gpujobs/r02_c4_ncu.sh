# C4 with the batched prior transform: launch list + one full capture of the advance kernel
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv \
  python bench.py --config c4 --steps 1 --warmup 3 --n 20 --no-cpu --no-lockstep > gpurun_out/r02_c4_ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fsm_advance_kernel -s 30 -c 1 \
  -o gpurun_out/r02_c4_advance python bench.py --config c4 --steps 1 --warmup 3 --n 20 --no-cpu --no-lockstep > gpurun_out/r02_c4_ncu_full.log 2>&1
tail -2 gpurun_out/r02_c4_ncu_full.log
