# round 2, first call: GPU suite after the ABI v4 change (per-state work words),
# bench-horizon parity reports, C2 bench
mkdir -p gpurun_out/r04a
export FSMC_HORIZON_OUT=gpurun_out/r04a
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r04a/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r04a/gpu_suite.log 2>&1; tail -3 gpurun_out/r04a/gpu_suite.log
grep -E "bit-exact over" gpurun_out/r04a/gpu_suite.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r04a/bench_c2.json 2> gpurun_out/r04a/bench_c2.err
tail -c 600 gpurun_out/r04a/bench_c2.json
