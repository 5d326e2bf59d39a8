timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prior or batched or lockstep" > gpurun_out/r02_pp_tests.log 2>&1; tail -1 gpurun_out/r02_pp_tests.log
for pp in 1 2 4; do timeout 300 python bench.py --config c4 --prior-parts $pp --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_pp_$pp.json 2> gpurun_out/r02_pp_$pp.err; tail -2 gpurun_out/r02_pp_$pp.err; done
