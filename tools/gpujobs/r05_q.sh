mkdir -p gpurun_out/r05q
for cfg in "8 4 15" "8 12 15" "8 16 15" "8 16 8" "32 16 15"; do set -- $cfg
  CUDA_DEVICE_MAX_CONNECTIONS=$1 FSMC_PART_STREAMS=$3 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $2 > gpurun_out/r05q/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05q/r.json').read().strip().splitlines()[-1]); print('q$1 p$2 s$3', '%.4g'%d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done
