# C2 e2e: progress checks every round vs every 2 rounds
mkdir -p gpurun_out/r05zn
for L in paper_2503_17405_b200/libfsmc.so variants/kc1/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/kc1/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r05zn/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zn/r.json').read().strip().splitlines()[-1]); print('$L', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['e2e']['ms'][1:], d['clocks']['sm_mhz'])"
done
