# round 2, call 5: hand-written DMMA prior transform (C4) -- tests, A/B against cuBLAS DTRMM,
# launch list; C2 source-level profiles of both hot kernels
mkdir -p gpurun_out/r04e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "prior" > gpurun_out/r04e/prior_tests.log 2>&1; tail -2 gpurun_out/r04e/prior_tests.log
for pr in dmma trmm; do timeout 600 python bench.py --config c4 --prior $pr --steps 3 --warmup 2 --no-cpu --no-lockstep > gpurun_out/r04e/c4_$pr.json 2> gpurun_out/r04e/c4_$pr.err; python -c "
import json; d=json.loads(open('gpurun_out/r04e/c4_$pr.json').read().strip().splitlines()[-1]); print('$pr', d['value'], d['ms_per_step'], d['e2e']['value'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04e/c4_launches.csv \
  python bench.py --config c4 --steps 1 --warmup 1 --n 20 --no-cpu --no-lockstep > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/r04e/c4_launches.csv 8
for k in drmh_draws_kernel fsm_window_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 \
    -o /tmp/r04e_$k python tools/issue_probe.py 200 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/r04e_$k.ncu-rep > gpurun_out/r04e/c2_$k.summary.txt 2>&1
  python tools/ncu_lines.py /tmp/r04e_$k.ncu-rep 60 > gpurun_out/r04e/c2_$k.lines.txt 2>&1
  ncu -i /tmp/r04e_$k.ncu-rep --page source --csv --print-source sass > /tmp/r04e_$k.sass.csv 2>/dev/null
  gzip -c /tmp/r04e_$k.sass.csv > gpurun_out/r04e/c2_$k.sass.csv.gz
done
ls gpurun_out/r04e
# generator with U slots per lane per pass (ILP) vs the previous one (variants/u1) and U=2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed or prng or overlapped" > gpurun_out/r04e/gen_tests.log 2>&1; tail -2 gpurun_out/r04e/gen_tests.log
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/u1/libfsmc.so variants/u2/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r04e/gen_ab.txt 2>&1; cat gpurun_out/r04e/gen_ab.txt
timeout 500 python -m pytest tests/test_gpu_sharded.py -q -x -rA -p no:cacheprovider > gpurun_out/r04e/sharded.log 2>&1; tail -40 gpurun_out/r04e/sharded.log | grep -v "^$" | tail -30
