# sincos in the elliptical proposal: device math test, ESS parity, C1 / C4 lines
mkdir -p gpurun_out/r05zc
export FSMC_HORIZON_OUT=gpurun_out/r05zc
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "device_math or ess or prior or c1 or c4" > gpurun_out/r05zc/tests.log 2>&1; tail -3 gpurun_out/r05zc/tests.log
for c in c1 c4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r05zc/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zc/r.json').read().strip().splitlines()[-1]); print('$c', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['roofline']['kernel_ms'])"
done
