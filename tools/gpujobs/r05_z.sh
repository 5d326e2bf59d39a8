# central-queue generator (FSMC_GEN_CQ): bit-exactness (windowed tests + C2 horizon) and A/B
mkdir -p gpurun_out/r05z
export FSMC_HORIZON_OUT=gpurun_out/r05z
FSMC_LIB=$(realpath variants/cq/libfsmc.so) timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider -k "windowed or c2 or smoke or normal" > gpurun_out/r05z/tests.log 2>&1; tail -3 gpurun_out/r05z/tests.log
bash tools/ab.sh "--steps 8 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/cq/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/cq/libfsmc.so > gpurun_out/r05z/ab.txt 2>&1
cat gpurun_out/r05z/ab.txt
