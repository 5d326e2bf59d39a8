mkdir -p gpurun_out/r05zi
bash tools/ab.sh "--config c3 --steps 4 --warmup 2 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/wmb4/libfsmc.so variants/wmb2/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r05zi/ab.txt 2>&1
cat gpurun_out/r05zi/ab.txt
