timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "lockstep or batched or prior" > gpurun_out/r02_lock_tests.log 2>&1
tail -3 gpurun_out/r02_lock_tests.log
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu > gpurun_out/r02_c5_lock.json 2> gpurun_out/r02_c5_lock.err
tail -3 gpurun_out/r02_c5_lock.err
