# round 2, call 7: straight-line tail queue in the draw generator (bit-exactness + A/B)
mkdir -p gpurun_out/r04g
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed or prng or overlapped" > gpurun_out/r04g/gen_tests.log 2>&1; tail -2 gpurun_out/r04g/gen_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c2" > gpurun_out/r04g/c2_horizon.log 2>&1; tail -2 gpurun_out/r04g/c2_horizon.log
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/tail0/libfsmc.so variants/u1/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r04g/gen_ab.txt 2>&1; cat gpurun_out/r04g/gen_ab.txt
timeout 300 ncu --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__cycles_active.avg --clock-control none \
  -k regex:"drmh_draws|fsm_window" --csv --log-file gpurun_out/r04g/c2_issue.csv python tools/issue_probe.py 200 > gpurun_out/r04g/c2_issue_probe.json 2> gpurun_out/r04g/c2_issue.err
python tools/issue_probe.py --summarise gpurun_out/r04g/c2_issue.csv gpurun_out/r04g/c2_issue_probe.json > gpurun_out/r04g/r04_c2_issue.json 2>&1
grep -A3 "by_kernel" gpurun_out/r04g/r04_c2_issue.json
