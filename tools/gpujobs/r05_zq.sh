# C2: small windows (draws L2-resident between generation and use)
mkdir -p gpurun_out/r05zq
for cfg in "8 4070" "8 1100" "8 2002" "16 1100" "8 660"; do set -- $cfg
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $1 --draw-window $2 > gpurun_out/r05zq/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zq/r.json').read().strip().splitlines()[-1]); print('p$1 W$2', '%.4g'%d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
