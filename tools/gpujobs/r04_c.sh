# round 2, call 3: fp16 operand variant of the fused C5 kernel, the distributional harness
mkdir -p gpurun_out/r04c
export FSMC_REPORT_OUT=gpurun_out/r04c
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused or tf32 or logreg" > gpurun_out/r04c/unit.log 2>&1; tail -2 gpurun_out/r04c/unit.log
for p in bf16-tc fp16-tc; do timeout 120 python tools/tc_probe.py 18944 $p 5; timeout 120 python tools/tc_probe.py 131072 $p 3; done > gpurun_out/r04c/tc_probe.txt 2>&1; cat gpurun_out/r04c/tc_probe.txt
timeout 1500 python -m pytest tests/test_gpu_distribution.py -q -rA -s -p no:cacheprovider > gpurun_out/r04c/dist.log 2>&1; grep -E "C5 shape|passed|failed|Error" gpurun_out/r04c/dist.log | tail -8
