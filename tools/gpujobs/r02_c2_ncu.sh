# full captures kept in /tmp on the box; summaries (text) come back in gpurun_out/
for k in drmh_draws_kernel fsm_window_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 \
    -o /tmp/r02_$k python bench.py --steps 1 --warmup 3 --n 200 --no-cpu --no-lockstep > gpurun_out/r02_c2_ncu_$k.log 2>&1
  python tools/ncu_summary.py /tmp/r02_$k.ncu-rep > gpurun_out/r02_c2_$k.summary.txt 2>&1
  python tools/ncu_lines.py /tmp/r02_$k.ncu-rep 60 > gpurun_out/r02_c2_$k.lines.txt 2>&1
  ncu -i /tmp/r02_$k.ncu-rep --page source --csv --print-source sass > /tmp/r02_$k.sass.csv 2>/dev/null
  gzip -c /tmp/r02_$k.sass.csv > gpurun_out/r02_c2_$k.sass.csv.gz
done
ls -la gpurun_out/
