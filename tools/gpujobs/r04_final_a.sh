# round 2 final (a): GPU suite, smoke, bench lines of every config, reference arm
mkdir -p gpurun_out/r04f_a
export FSMC_HORIZON_OUT=gpurun_out/r04f_a FSMC_REPORT_OUT=gpurun_out/r04f_a
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r04f_a/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r04f_a/gpu_suite.log 2>&1; grep -E "passed|failed" gpurun_out/r04f_a/gpu_suite.log | tail -2
grep -E "bit-exact over|C5 shape|fp32 vs" gpurun_out/r04f_a/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04f_a/smoke.log 2>&1; tail -1 gpurun_out/r04f_a/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r04f_a/bench_c2.json 2> gpurun_out/r04f_a/bench_c2.err; tail -c 400 gpurun_out/r04f_a/bench_c2.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r04f_a/bench_c2_reference.json 2>&1
for c in c1 c3 c4 c2f c3f; do timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r04f_a/bench_$c.json 2> gpurun_out/r04f_a/bench_$c.err; done
timeout 2400 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r04f_a/bench_c5.json 2> gpurun_out/r04f_a/bench_c5.err
for c in c2 c1 c3 c4 c2f c3f c5; do python -c "
import json; d=json.loads(open('gpurun_out/r04f_a/bench_$c.json').read().strip().splitlines()[-1]); print('$c', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%d['roofline']['frac'], 'lock', (d.get('lockstep') or {}).get('speedup'), d['clocks'])" 2>&1 | tail -1; done
