mkdir -p gpurun_out/r05zk
for c in c3 c3f c5; do
  timeout 2000 python bench.py --config $c --steps $([ $c = c5 ] && echo 2 || echo 4) --warmup $([ $c = c5 ] && echo 2 || echo 3) --no-cpu --no-lockstep > gpurun_out/r05zk/bench_$c.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05zk/bench_$c.json').read().strip().splitlines()[-1]); print('$c', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
