# C2 under bounded generators: window size and part count
mkdir -p gpurun_out/r05zg
for cfg in "8 4070" "8 3003" "8 6006" "8 8140" "6 4070" "10 4070" "12 4070" "8 4070"; do set -- $cfg
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --draw-parts $1 --draw-window $2 > gpurun_out/r05zg/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zg/r.json').read().strip().splitlines()[-1]); print('p$1 W$2', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
