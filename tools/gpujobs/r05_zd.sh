# C3 e2e: chain parts of the per-chain run with host output
mkdir -p gpurun_out/r05zd
for cfg in "2048 8" "1024 16" "4096 4" "1024 12"; do set -- $cfg
  FSMC_EGRESS_PART_CHAINS=$1 FSMC_EGRESS_PARTS_MAX=$2 timeout 600 python bench.py --config c3 --steps 4 --warmup 2 --no-cpu --no-lockstep > gpurun_out/r05zd/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zd/r.json').read().strip().splitlines()[-1]); print('c3 chains$1 max$2', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['e2e']['ms'][1:])"
done
