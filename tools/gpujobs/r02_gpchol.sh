timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gp" > gpurun_out/r02_gpchol_tests.log 2>&1
tail -3 gpurun_out/r02_gpchol_tests.log
timeout 900 python tools/paper_gp_experiment.py 200 1 128 1024 > gpurun_out/r02_paper_gp_200b.json 2> gpurun_out/r02_paper_gpb.err
tail -4 gpurun_out/r02_paper_gpb.err
