# round 2, call 8: generator variants A/B (tail queue forms, occupancy)
mkdir -p gpurun_out/r04h
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed or prng or overlapped or wide" > gpurun_out/r04h/tests.log 2>&1; tail -2 gpurun_out/r04h/tests.log
for L in paper_2503_17405_b200/libfsmc.so variants/tail0/libfsmc.so variants/tail2/libfsmc.so variants/occ5/libfsmc.so variants/occ6/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed_draws_are_bit" > /dev/null 2>&1 && echo "$L bit-exact" || echo "$L MISMATCH"
done
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/tail0/libfsmc.so variants/tail2/libfsmc.so variants/occ5/libfsmc.so variants/occ6/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r04h/gen_ab.txt 2>&1; cat gpurun_out/r04h/gen_ab.txt
