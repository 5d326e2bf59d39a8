mkdir -p gpurun_out/r05zv
bash tools/ab.sh "--config c3 --steps 4 --warmup 2 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/tickc/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/tickc/libfsmc.so > gpurun_out/r05zv/ab.txt 2>&1; cat gpurun_out/r05zv/ab.txt
