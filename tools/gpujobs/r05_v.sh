# C4 prior parts sweep (32 hardware queues)
mkdir -p gpurun_out/r05v
for P in 1 2 3 4 6 8; do
  timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu --no-lockstep --prior-parts $P > gpurun_out/r05v/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05v/r.json').read().strip().splitlines()[-1]); print('c4 p$P', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'])"
done
