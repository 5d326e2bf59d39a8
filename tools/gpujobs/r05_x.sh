# C4: prior rounds issued without host waits (counts read one round late): tests + parts sweep
mkdir -p gpurun_out/r05x
export FSMC_HORIZON_OUT=gpurun_out/r05x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "prior or c4 or streamed" > gpurun_out/r05x/tests.log 2>&1; tail -3 gpurun_out/r05x/tests.log
for P in 1 2 3 4 6; do
  timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu --no-lockstep --prior-parts $P > gpurun_out/r05x/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05x/r.json').read().strip().splitlines()[-1]); print('c4 p$P', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'])"
done
