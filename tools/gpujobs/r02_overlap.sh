timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed" > gpurun_out/r02_ov_tests.log 2>&1
tail -2 gpurun_out/r02_ov_tests.log
for pp in 1 2; do timeout 300 python bench.py --draw-parts $pp --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_ov_$pp.json 2> gpurun_out/r02_ov_$pp.err; tail -2 gpurun_out/r02_ov_$pp.err; done
