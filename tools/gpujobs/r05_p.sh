# C2: chain parts sharing FSMC_PART_STREAMS streams (32 hardware queues): value and e2e
mkdir -p gpurun_out/r05p
for cfg in "32 16 8" "32 16 4" "32 12 6" "32 12 4" "32 8 4" "32 16 6" "8 16 8" "32 16 16" "32 16 8"; do set -- $cfg
  CUDA_DEVICE_MAX_CONNECTIONS=$1 FSMC_PART_STREAMS=$3 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --draw-parts $2 > gpurun_out/r05p/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05p/r.json').read().strip().splitlines()[-1]); print('q$1 p$2 s$3', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'])"
done > gpurun_out/r05p/matrix.txt 2>&1
cat gpurun_out/r05p/matrix.txt
