# plain / amortized executor specialised per state (tick VAR 2): parity + C1 A/B
mkdir -p gpurun_out/r05zs
export FSMC_HORIZON_OUT=gpurun_out/r05zs
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "golden or c1 or amortized or plain or ess or drmh or slice or smoke" > gpurun_out/r05zs/tests.log 2>&1; tail -1 gpurun_out/r05zs/tests.log
for L in paper_2503_17405_b200/libfsmc.so variants/novar2/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/novar2/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 600 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zs/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zs/r.json').read().strip().splitlines()[-1]); print('$L', '%.4g'%d['value'], d['roofline']['kernel_ms'])"
done
