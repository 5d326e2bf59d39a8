# 32 hardware queues: bounded generators in flight (FSMC_GEN_SLOTS) x parts
mkdir -p gpurun_out/r05s
for cfg in "12 0" "12 4" "12 6" "12 8" "14 6" "14 8" "8 4" "15 8" "12 3"; do set -- $cfg
  CUDA_DEVICE_MAX_CONNECTIONS=32 FSMC_GEN_SLOTS=$2 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $1 > gpurun_out/r05s/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05s/r.json').read().strip().splitlines()[-1]); print('q32 p$1 slots$2', '%.4g'%d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done
