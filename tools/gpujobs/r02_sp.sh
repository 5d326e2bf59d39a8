timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_sp_suite.log 2>&1
tail -2 gpurun_out/r02_sp_suite.log
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/r02_sp_$c.json 2> gpurun_out/r02_sp_$c.err; done
