# math.exp restated (gl_exp) at the DRMH accept / NUTS sites, MoG exp variants; race fix for the
# batched prior rounds (chain-owned rows) and the evaluator rounds (no theta read-back)
mkdir -p gpurun_out/r05c
export FSMC_HORIZON_OUT=gpurun_out/r05c FSMC_REPORT_OUT=gpurun_out/r05c
bash tools/ab.sh "--steps 8 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/glmog/libfsmc.so variants/cudaexp/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r05c/ab.txt 2>&1
cat gpurun_out/r05c/ab.txt
bash tools/ab.sh "--config c3 --steps 4 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/cudaexp3/libfsmc.so > gpurun_out/r05c/ab_c3.txt 2>&1
cat gpurun_out/r05c/ab_c3.txt
timeout 600 python bench.py --config c4 --steps 4 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r05c/bench_c4.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r05c/bench_c4.json').read().strip().splitlines()[-1]); print('c4', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r05c/gpu_suite.log 2>&1; tail -3 gpurun_out/r05c/gpu_suite.log
grep -E "bit-exact over" gpurun_out/r05c/gpu_suite.log
