# 32 hardware work queues (package default) vs CUDA's 8: C2 value + e2e, C3/C4 lines
mkdir -p gpurun_out/r05n
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['e2e']['ms'][1:], d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1 $2; }
for Q in 32 8; do
  CUDA_DEVICE_MAX_CONNECTIONS=$Q timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r05n/c2_q$Q.json 2>/dev/null; line gpurun_out/r05n/c2_q$Q.json "c2 q$Q"
done
for c in c3 c4; do for Q in 32 8; do
  CUDA_DEVICE_MAX_CONNECTIONS=$Q timeout 900 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r05n/${c}_q$Q.json 2>/dev/null; line gpurun_out/r05n/${c}_q$Q.json "$c q$Q"
done; done
