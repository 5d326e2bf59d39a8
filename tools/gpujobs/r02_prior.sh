timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prior" > gpurun_out/r02_prior_tests.log 2>&1
tail -3 gpurun_out/r02_prior_tests.log
for pr in none gemm device; do timeout 300 python bench.py --config c4 --prior $pr --steps 2 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_c4_$pr.json 2> gpurun_out/r02_c4_$pr.err; tail -2 gpurun_out/r02_c4_$pr.err; done
