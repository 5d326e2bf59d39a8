# every bench line at HEAD with the e2e rule (>= 3 warm-ups, mean over timed calls) and the r06 C2 traffic capture
mkdir -p gpurun_out/r06c
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r06c/bench_c2.json 2> gpurun_out/r06c/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r06c/bench_c2_reference.json 2>&1
for c in c1 c3 c4 c2f c3f; do timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r06c/bench_$c.json 2> gpurun_out/r06c/bench_$c.err; done
timeout 2400 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r06c/bench_c5.json 2> gpurun_out/r06c/bench_c5.err
python tools/bench_table.py gpurun_out/r06c
