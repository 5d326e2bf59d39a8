# round 2, call 9: generator with the straight-line tail: ILP width and occupancy variants
mkdir -p gpurun_out/r04i
for L in paper_2503_17405_b200/libfsmc.so variants/u2/libfsmc.so variants/u8/libfsmc.so variants/m3/libfsmc.so variants/m4/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed_draws_are_bit" > /dev/null 2>&1 && echo "$L bit-exact" || echo "$L MISMATCH"
done
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/u2/libfsmc.so variants/u8/libfsmc.so variants/m3/libfsmc.so variants/m4/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r04i/gen_ab.txt 2>&1; cat gpurun_out/r04i/gen_ab.txt
