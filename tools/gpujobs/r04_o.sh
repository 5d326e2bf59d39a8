# round 2: user-defined batched targets; bench's multi-rank path on one GPU (gloo)
mkdir -p gpurun_out/r04o
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "user_batched or gp or errors" > gpurun_out/r04o/user.log 2>&1; tail -3 gpurun_out/r04o/user.log
timeout 1200 python -m pytest tests/test_gpu_bench_multirank.py -q -x -p no:cacheprovider > gpurun_out/r04o/multirank.log 2>&1; tail -15 gpurun_out/r04o/multirank.log
