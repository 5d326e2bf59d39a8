# NVTX ranges in the C ABI: C2 line unchanged, windowed / prior tests, and ncu sees the ranges
mkdir -p gpurun_out/r05zr
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider -k "windowed or prior or streamed" > gpurun_out/r05zr/tests.log 2>&1; tail -1 gpurun_out/r05zr/tests.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05zr/r.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r05zr/r.json').read().strip().splitlines()[-1]); print('c2', '%.4g'%d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
timeout 600 ncu --nvtx --nvtx-include "fsmc_run_windowed_egress/" --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/r05zr/nvtx_launches.csv python bench.py --steps 1 --warmup 0 --samples 20 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"; grep -c "drmh_draws\|fsm_window" gpurun_out/r05zr/nvtx_launches.csv
