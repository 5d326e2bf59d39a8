timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or prng" > gpurun_out/r02_c2a_tests.log 2>&1
tail -2 gpurun_out/r02_c2a_tests.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_c2a.json 2> gpurun_out/r02_c2a.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c2a_launches.csv \
  python bench.py --steps 1 --warmup 3 --n 200 --no-cpu --no-lockstep > /dev/null 2>&1
