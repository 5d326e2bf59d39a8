# C2: hardware work queues x chain parts, device value and e2e (host output)
mkdir -p gpurun_out/r05o
for Q in 8 16 32; do for P in 4 6 7 8 12 16; do
  CUDA_DEVICE_MAX_CONNECTIONS=$Q timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --draw-parts $P > gpurun_out/r05o/q${Q}_p$P.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05o/q${Q}_p$P.json').read().strip().splitlines()[-1]); print('q$Q p$P', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'])"
done; done > gpurun_out/r05o/matrix.txt 2>&1
cat gpurun_out/r05o/matrix.txt
