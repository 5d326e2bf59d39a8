# advance_chain specialised per state (non-bundled): GPU suite + C4 / C1 A/B
mkdir -p gpurun_out/r05zt
export FSMC_HORIZON_OUT=gpurun_out/r05zt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r05zt/tests.log 2>&1; tail -1 gpurun_out/r05zt/tests.log
for L in paper_2503_17405_b200/libfsmc.so variants/novar2/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/novar2/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zt/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zt/r.json').read().strip().splitlines()[-1]); print('c4 $L', '%.4g'%d['value'], d['roofline']['kernel_ms'])"
done
