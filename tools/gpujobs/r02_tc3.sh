timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05 or logreg or fused" > gpurun_out/r02_tc3_tests.log 2>&1
tail -1 gpurun_out/r02_tc3_tests.log
for r in 1 2; do timeout 300 python tools/tc_probe.py 131072 bf16-tc 5 >> gpurun_out/r02_tc3_probe.txt 2>&1; done
