# glibc exp restated on the device (gl_exp) vs CUDA's exp: C2 A/B, then the GPU suite
mkdir -p gpurun_out/r05b
export FSMC_HORIZON_OUT=gpurun_out/r05b FSMC_REPORT_OUT=gpurun_out/r05b
bash tools/ab.sh "--steps 8 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/cudaexp/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/cudaexp/libfsmc.so > gpurun_out/r05b/ab.txt 2>&1
cat gpurun_out/r05b/ab.txt
for c in c3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05b/bench_$c.json 2>/dev/null; tail -c 300 gpurun_out/r05b/bench_$c.json; echo; done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r05b/gpu_suite.log 2>&1; tail -3 gpurun_out/r05b/gpu_suite.log
grep -E "bit-exact over" gpurun_out/r05b/gpu_suite.log
