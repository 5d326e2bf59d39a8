# round 2 (session 2): window-kernel prefetch depth and the software-pipelined generator, A/B
mkdir -p gpurun_out/r05a
bash tools/ab.sh "--steps 8 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/pf2/libfsmc.so variants/pf3/libfsmc.so variants/pipe/libfsmc.so variants/pipe4/libfsmc.so variants/pipepf2/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r05a/ab.txt 2>&1
cat gpurun_out/r05a/ab.txt
