mkdir -p gpurun_out/r05za
for L in 128 32; do
  timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --no-lockstep --lanes $L > gpurun_out/r05za/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05za/r.json').read().strip().splitlines()[-1]); print('c1 lanes$L', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['roofline']['kernel_ms'], d['ms_per_step'])"
done
