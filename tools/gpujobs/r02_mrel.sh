timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_mrel_suite.log 2>&1; tail -1 gpurun_out/r02_mrel_suite.log
for r in 1 2; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_mrel_$r.json 2>/dev/null; done
