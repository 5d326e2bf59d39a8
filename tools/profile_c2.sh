#!/bin/bash
# On the GPU box: headline bench line, launch list and a full ncu capture of
# the DRMH step kernel.  Outputs land in gpurun_out/ (copy summaries to profiles/).
set -x
timeout 900 python bench.py > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
echo bench=$?
CMD="python bench.py --steps 2 --warmup 3 --n 200 --no-cpu --no-lockstep"
$CMD > gpurun_out/launch_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/launch_ncu.log 2>&1
echo launches=$?
CMD2="python bench.py --steps 1 --warmup 1 --n 200 --no-cpu --no-lockstep"
$CMD2 > gpurun_out/full_plain.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsm_run_kernel \
    -s 1 -c 1 -o gpurun_out/prof_c2 $CMD2 > gpurun_out/full_ncu.log 2>&1
echo full=$?
