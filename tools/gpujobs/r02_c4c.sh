timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prior" > gpurun_out/r02_c4c_tests.log 2>&1
tail -3 gpurun_out/r02_c4c_tests.log
for pr in trmm; do timeout 300 python bench.py --config c4 --prior $pr --steps 3 --warmup 3 --no-cpu > gpurun_out/r02c_c4_$pr.json 2> gpurun_out/r02c_c4_$pr.err; tail -2 gpurun_out/r02c_c4_$pr.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_c4_launches.csv \
  python bench.py --config c4 --prior trmm --steps 1 --warmup 3 --n 20 --no-cpu --no-lockstep > /dev/null 2>&1
