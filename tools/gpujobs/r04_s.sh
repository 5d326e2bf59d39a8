# round 2: int64 count matrices streamed with the samples (ABI 6)
mkdir -p gpurun_out/r04s
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider > gpurun_out/r04s/tests.log 2>&1; tail -1 gpurun_out/r04s/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r04s/bench.json 2> gpurun_out/r04s/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r04s/bench.json').read().strip().splitlines()[-1]); print(d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms'], d['e2e']['d2h_bytes_per_step'])"
timeout 600 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu --no-lockstep > gpurun_out/r04s/bench_c3.json 2> gpurun_out/r04s/bench_c3.err; python -c "
import json; d=json.loads(open('gpurun_out/r04s/bench_c3.json').read().strip().splitlines()[-1]); print('c3', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms'])"
