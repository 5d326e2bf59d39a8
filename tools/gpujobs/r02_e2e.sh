timeout 600 python tools/e2e_breakdown.py c2 > gpurun_out/r02_e2e_c2.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c1 > gpurun_out/r02_e2e_c1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ess" > gpurun_out/r02_e2e_tests.log 2>&1
tail -1 gpurun_out/r02_e2e_tests.log
