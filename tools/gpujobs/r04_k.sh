# round 2, call 11: DRMH candidate in place + exact-dimension benchmark kernels
mkdir -p gpurun_out/r04k
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider > gpurun_out/r04k/tests.log 2>&1; tail -2 gpurun_out/r04k/tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c2" > gpurun_out/r04k/c2_horizon.log 2>&1; tail -1 gpurun_out/r04k/c2_horizon.log
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r04k/ab.txt 2>&1; cat gpurun_out/r04k/ab.txt
