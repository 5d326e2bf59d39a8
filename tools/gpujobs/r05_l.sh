# per-part sample egress (windowed runs): tests, then the C2 line (e2e) at 12 and 4 parts
mkdir -p gpurun_out/r05l
timeout 900 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "streamed or windowed" > gpurun_out/r05l/tests.log 2>&1; tail -3 gpurun_out/r05l/tests.log
for P in 12 4 16; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-lockstep --draw-parts $P > gpurun_out/r05l/bench_p$P.json 2> gpurun_out/r05l/bench_p$P.err; python -c "
import json; d=json.loads(open('gpurun_out/r05l/bench_p$P.json').read().strip().splitlines()[-1]); print('p$P', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['e2e']['ms'], d['clocks'])"; done
