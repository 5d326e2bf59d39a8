# bounded generators: value and e2e
mkdir -p gpurun_out/r05t
for cfg in "8 4" "12 4" "12 6" "6 3" "4 2" "8 2" "16 4"; do set -- $cfg
  FSMC_GEN_SLOTS=$2 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --draw-parts $1 > gpurun_out/r05t/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05t/r.json').read().strip().splitlines()[-1]); print('p$1 slots$2', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['e2e']['ms'][1:], d['clocks']['sm_mhz'])"
done
