mkdir -p gpurun_out/r05zl
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "nuts or c3 or fp32 or race" > gpurun_out/r05zl/tests.log 2>&1; tail -2 gpurun_out/r05zl/tests.log
for c in c3 c3f; do
  timeout 2000 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zl/bench_$c.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zl/bench_$c.json').read().strip().splitlines()[-1]); print('$c', '%.4g'%d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
