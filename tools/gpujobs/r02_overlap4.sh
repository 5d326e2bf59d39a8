timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed" > gpurun_out/r02_ov4_tests.log 2>&1
tail -2 gpurun_out/r02_ov4_tests.log
for pp in 2 3 4; do timeout 300 python bench.py --draw-parts $pp --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_ovp_$pp.json 2> gpurun_out/r02_ovp_$pp.err; done
