# round 2, call 2: new tests (concurrency, horizons at 128 chains), bench C2 with the
# host-output e2e + lock-step accounting, C2 issue counts
mkdir -p gpurun_out/r04b
timeout 900 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r04b/tests.log 2>&1; tail -3 gpurun_out/r04b/tests.log
timeout 300 ncu --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__cycles_active.avg --clock-control none \
  -k regex:"drmh_draws|fsm_window" --csv --log-file gpurun_out/r04b/c2_issue.csv python tools/issue_probe.py 200 > gpurun_out/r04b/c2_issue_probe.json 2> gpurun_out/r04b/c2_issue.err
python tools/issue_probe.py --summarise gpurun_out/r04b/c2_issue.csv gpurun_out/r04b/c2_issue_probe.json > gpurun_out/r04b/r04_c2_issue.json 2>&1
cp gpurun_out/r04b/r04_c2_issue.json profiles/ 2>/dev/null
head -c 600 gpurun_out/r04b/r04_c2_issue.json
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r04b/bench_c2.json 2> gpurun_out/r04b/bench_c2.err
tail -3 gpurun_out/r04b/bench_c2.err
python -c "
import json; d=json.loads(open('gpurun_out/r04b/bench_c2.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e'], 'e2e_dev', d['e2e_device']['value'])
print('lock', json.dumps(d['lockstep']))
print('roof', d['roofline']['frac'], d['roofline'].get('issue'))
"
