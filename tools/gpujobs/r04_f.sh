# round 2, call 6: sharded runs, DMMA prior transform v2 (64x64 tiles) vs cuBLAS, fp32 throughput mode
mkdir -p gpurun_out/r04f
export FSMC_REPORT_OUT=gpurun_out/r04f
timeout 500 python -m pytest tests/test_gpu_sharded.py -q -x -rA -p no:cacheprovider > gpurun_out/r04f/sharded.log 2>&1; grep -E "passed|failed|Error" gpurun_out/r04f/sharded.log | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "prior" > gpurun_out/r04f/prior_tests.log 2>&1; tail -1 gpurun_out/r04f/prior_tests.log
for pr in dmma trmm; do timeout 600 python bench.py --config c4 --prior $pr --steps 3 --warmup 2 --no-cpu --no-lockstep --no-e2e > gpurun_out/r04f/c4_$pr.json 2> gpurun_out/r04f/c4_$pr.err; python -c "
import json; d=json.loads(open('gpurun_out/r04f/c4_$pr.json').read().strip().splitlines()[-1]); print('$pr', d['value'], d['ms_per_step'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04f/c4_launches.csv \
  python bench.py --config c4 --steps 1 --warmup 1 --n 20 --no-cpu --no-lockstep --no-e2e > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/r04f/c4_launches.csv 4
timeout 900 python -m pytest tests/test_gpu_distribution.py -q -s -rA -p no:cacheprovider -k "fp32" > gpurun_out/r04f/fp32.log 2>&1; grep -E "fp32 vs|passed|failed" gpurun_out/r04f/fp32.log | tail -4
for c in c2f c3f; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-lockstep > gpurun_out/r04f/bench_$c.json 2> gpurun_out/r04f/bench_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/r04f/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'])"; done
