timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_suite.log 2>&1
tail -2 gpurun_out/r02_gpu_suite.log
for c in c1 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; done
k=fsm_run_kernel
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 \
    -o /tmp/r02_c3 python bench.py --config c3 --steps 1 --warmup 3 --n 100 --no-cpu --no-lockstep > gpurun_out/r02_c3_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r02_c3.ncu-rep > gpurun_out/r02_c3.summary.txt 2>&1
python tools/ncu_lines.py /tmp/r02_c3.ncu-rep 60 > gpurun_out/r02_c3.lines.txt 2>&1
