mkdir -p gpurun_out/r05zw
export FSMC_HORIZON_OUT=gpurun_out/r05zw
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "nuts or c3 or fp32" > gpurun_out/r05zw/tests.log 2>&1; tail -1 gpurun_out/r05zw/tests.log
for c in c3 c3f; do timeout 600 python bench.py --config $c --steps 4 --warmup 2 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zw/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zw/r.json').read().strip().splitlines()[-1]); print('$c', '%.4g'%d['value'], d['roofline']['kernel_ms'])"; done
