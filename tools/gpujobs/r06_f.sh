# last pass at HEAD: GPU suite, smoke, the C2 headline line and the lines whose roofline.traffic source changed
mkdir -p gpurun_out/r06f
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r06f/gpu_suite.log 2>&1; tail -1 gpurun_out/r06f/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r06f/smoke.log 2>&1; tail -1 gpurun_out/r06f/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r06f/bench_c2.json 2> gpurun_out/r06f/bench_c2.err
for c in c1 c3 c4; do timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r06f/bench_$c.json 2> gpurun_out/r06f/bench_$c.err; done
python tools/bench_table.py gpurun_out/r06f
