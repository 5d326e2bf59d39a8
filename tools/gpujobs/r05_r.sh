# 32 hardware queues: generator grid caps x parts (value only)
mkdir -p gpurun_out/r05r
for cfg in "12 1 0" "12 2 0" "16 1 0" "8 1 0" "12 1 1" "16 2 1" "12 4 0" "16 1 1"; do set -- $cfg
  CUDA_DEVICE_MAX_CONNECTIONS=32 FSMC_PART_STREAMS=15 FSMC_DRAW_BLOCKS_PER_SM=$2 FSMC_WIN_BLOCKS_PER_SM=$3 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $1 > gpurun_out/r05r/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05r/r.json').read().strip().splitlines()[-1]); print('q32 p$1 g$2 w$3', '%.4g'%d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done
