# round 2, call 10: GP gradient kernel (tests + launch list of the NUTS GP run), generator u2 vs u4
mkdir -p gpurun_out/r04j
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gp" > gpurun_out/r04j/gp_tests.log 2>&1; tail -3 gpurun_out/r04j/gp_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gp_batched_runs_match_oracle and nuts" > gpurun_out/r04j/gp_nuts_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04j/gp_nuts_launches.csv \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gp_batched_runs_match_oracle and nuts" > gpurun_out/r04j/gp_nuts_ncu.log 2>&1
python tools/launch_shares.py gpurun_out/r04j/gp_nuts_launches.csv 12
grep -ci "cusolver\|potrf\|potrs\|trsm\|syrk\|getrf" gpurun_out/r04j/gp_nuts_launches.csv
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/u2/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/u2/libfsmc.so > gpurun_out/r04j/gen_ab.txt 2>&1; cat gpurun_out/r04j/gen_ab.txt
