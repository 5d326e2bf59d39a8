# round 2: non-draining progress checks in the windowed run
mkdir -p gpurun_out/r04r
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider -k "windowed or overlapped or concurren or streamed or errors" > gpurun_out/r04r/tests.log 2>&1; tail -1 gpurun_out/r04r/tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c2" > gpurun_out/r04r/c2.log 2>&1; tail -1 gpurun_out/r04r/c2.log
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r04r/ab.txt 2>&1; cat gpurun_out/r04r/ab.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r04r/bench.json 2> gpurun_out/r04r/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r04r/bench.json').read().strip().splitlines()[-1]); print(d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms'])"
