k=fsm_advance_kernel
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 30 -c 1 \
    -o /tmp/r02_c4b python bench.py --config c4 --steps 1 --warmup 3 --n 20 --no-cpu --no-lockstep > gpurun_out/r02_c4b_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r02_c4b.ncu-rep > gpurun_out/r02_c4b.summary.txt 2>&1
python tools/ncu_lines.py /tmp/r02_c4b.ncu-rep 50 > gpurun_out/r02_c4b.lines.txt 2>&1
