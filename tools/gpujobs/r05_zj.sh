# NUTS trajectory ends in shared memory: parity (NUTS goldens, C3 horizon, batched rounds) and C3 / C5 A/B
mkdir -p gpurun_out/r05zj
export FSMC_HORIZON_OUT=gpurun_out/r05zj
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "nuts or c3 or c5 or race or sharded or concurrency or distribution" > gpurun_out/r05zj/tests.log 2>&1; tail -3 gpurun_out/r05zj/tests.log
bash tools/ab.sh "--config c3 --steps 4 --warmup 2 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/nutsreg/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/nutsreg/libfsmc.so > gpurun_out/r05zj/ab.txt 2>&1
cat gpurun_out/r05zj/ab.txt
