# round 2, call 12: streamed host output of the per-chain run (fsmc_run_egress)
mkdir -p gpurun_out/r04l
timeout 900 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r04l/tests.log 2>&1; tail -2 gpurun_out/r04l/tests.log
for c in c3 c1; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-lockstep > gpurun_out/r04l/bench_$c.json 2> gpurun_out/r04l/bench_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/r04l/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['ms'], 'dev', d['e2e_device']['value'])"; done
