# C4: softplus with glibc's table exp (FSMC_SP_GLEXP) A/B, plus the C4 horizon test on the variant
mkdir -p gpurun_out/r05zp
export FSMC_HORIZON_OUT=gpurun_out/r05zp
FSMC_LIB=$(realpath variants/spgl/libfsmc.so) timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c4 or gpc or prior or ess" > gpurun_out/r05zp/tests.log 2>&1; tail -2 gpurun_out/r05zp/tests.log
for L in paper_2503_17405_b200/libfsmc.so variants/spgl/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/spgl/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zp/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zp/r.json').read().strip().splitlines()[-1]); print('$L', '%.4g'%d['value'], d['roofline']['kernel_ms'])"
done
