for pp in 4 6 8; do timeout 300 python bench.py --draw-parts $pp --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_p8_$pp.json 2> gpurun_out/r02_p8_$pp.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed" > gpurun_out/r02_p8_tests.log 2>&1; tail -1 gpurun_out/r02_p8_tests.log
