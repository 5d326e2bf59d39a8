# C3 run kernel: one ncu --set full capture (n = 100)
mkdir -p gpurun_out/r05zh
timeout 300 python bench.py --config c3 --n 100 --steps 1 --warmup 1 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"fsm_run_kernel" -c 1 \
  -o gpurun_out/r05zh/c3_run python bench.py --config c3 --n 100 --steps 1 --warmup 0 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zh/ncu.log 2>&1
ls -la gpurun_out/r05zh/
