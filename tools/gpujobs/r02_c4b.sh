timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prior or gpc or gp_classification or batched or lane" > gpurun_out/r02_c4b_tests.log 2>&1
tail -3 gpurun_out/r02_c4b_tests.log
for pr in none gemm; do timeout 300 python bench.py --config c4 --prior $pr --steps 2 --warmup 3 --no-cpu > gpurun_out/r02b_c4_$pr.json 2> gpurun_out/r02b_c4_$pr.err; tail -2 gpurun_out/r02b_c4_$pr.err; done
timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu > gpurun_out/r02b_c5.json 2> gpurun_out/r02b_c5.err
