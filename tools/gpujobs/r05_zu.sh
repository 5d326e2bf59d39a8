mkdir -p gpurun_out/r05zu
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "prior or batched or lockstep or gp or logreg or race or c4" > gpurun_out/r05zu/tests.log 2>&1; tail -1 gpurun_out/r05zu/tests.log
for c in c4 c1; do timeout 600 python bench.py --config $c --steps 4 --warmup 2 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zu/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zu/r.json').read().strip().splitlines()[-1]); print('$c', '%.4g'%d['value'], d['roofline']['kernel_ms'])"; done
