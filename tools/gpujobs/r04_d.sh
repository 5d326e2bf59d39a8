# round 2, call 4: C5 distributional harness at a longer horizon (+ fp64 control);
# sharded runs on one GPU (two gloo ranks, no cross-rank waits inside kernels)
mkdir -p gpurun_out/r04d
export FSMC_REPORT_OUT=gpurun_out/r04d
timeout 1500 python -m pytest tests/test_gpu_distribution.py -q -rA -s -p no:cacheprovider > gpurun_out/r04d/dist.log 2>&1; grep -E "C5 shape|passed|failed|Error|xfail" gpurun_out/r04d/dist.log | tail -8
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -rA -p no:cacheprovider > gpurun_out/r04d/sharded.log 2>&1; tail -5 gpurun_out/r04d/sharded.log
