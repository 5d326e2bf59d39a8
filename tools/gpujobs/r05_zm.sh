# C4 advance kernel: one ncu --set full capture
mkdir -p gpurun_out/r05zm
timeout 300 python bench.py --config c4 --n 10 --steps 1 --warmup 1 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"fsm_advance_kernel" -s 6 -c 1 \
  -o gpurun_out/r05zm/c4_adv python bench.py --config c4 --n 10 --steps 1 --warmup 0 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zm/ncu.log 2>&1
ls -la gpurun_out/r05zm/
