# device math test; three-IMAD 64-bit multiply in the generator hash (A/B)
mkdir -p gpurun_out/r05g
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "device_math or windowed or prior_rounds or normal" > gpurun_out/r05g/tests.log 2>&1; tail -3 gpurun_out/r05g/tests.log
bash tools/ab.sh "--steps 8 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/mul3/libfsmc.so paper_2503_17405_b200/libfsmc.so variants/mul3/libfsmc.so > gpurun_out/r05g/ab.txt 2>&1
cat gpurun_out/r05g/ab.txt
