# round 2, call: window-kernel trims (constant-state bookkeeping, tick count per window,
# K-1 MoG exponentials) A/B; C4 streamed host output
mkdir -p gpurun_out/r04n
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider > gpurun_out/r04n/tests.log 2>&1; tail -2 gpurun_out/r04n/tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c2" > gpurun_out/r04n/c2_horizon.log 2>&1; tail -1 gpurun_out/r04n/c2_horizon.log
for L in variants/nt0/libfsmc.so variants/tc0/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed_draws or mog10" > /dev/null 2>&1 && echo "$L ok" || echo "$L FAIL"
done
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/nt0/libfsmc.so variants/tc0/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r04n/ab.txt 2>&1; cat gpurun_out/r04n/ab.txt
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu --no-lockstep > gpurun_out/r04n/bench_c4.json 2> gpurun_out/r04n/bench_c4.err; python -c "
import json; d=json.loads(open('gpurun_out/r04n/bench_c4.json').read().strip().splitlines()[-1]); print('c4', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms'])"
