# f4: kernels launched by NUTS on the GP-hyperparameter target (batched evaluator, n_obs = 90 and 414)
mkdir -p gpurun_out/r05zo
for N in 90 414; do
  timeout 300 python tools/gp_nuts_launches.py $N > gpurun_out/r05zo/plain_$N.txt 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r05zo/launches_$N.csv python tools/gp_nuts_launches.py $N > gpurun_out/r05zo/ncu_$N.txt 2>&1
  python tools/launch_shares.py gpurun_out/r05zo/launches_$N.csv 20 > gpurun_out/r05zo/shares_$N.md
  cat gpurun_out/r05zo/plain_$N.txt; cat gpurun_out/r05zo/shares_$N.md
done
