timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_e2e2_suite.log 2>&1
tail -1 gpurun_out/r02_e2e2_suite.log
timeout 600 python tools/e2e_breakdown.py c2 > gpurun_out/r02_e2e2_c2.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c1 > gpurun_out/r02_e2e2_c1.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/r02_e2e2_c3.txt 2>&1
