for r in 1 2; do
timeout 300 python tools/tc_probe.py 131072 bf16-tc 5 >> gpurun_out/r02_tc_ab.txt 2>&1
cp paper_2503_17405_b200/libfsmc.so /tmp/new.so; cp variants_tmp/libfsmc_before.so paper_2503_17405_b200/libfsmc.so
echo "old:" >> gpurun_out/r02_tc_ab.txt
timeout 300 python tools/tc_probe.py 131072 bf16-tc 5 >> gpurun_out/r02_tc_ab.txt 2>&1
cp /tmp/new.so paper_2503_17405_b200/libfsmc.so
echo "new:" >> gpurun_out/r02_tc_ab.txt
done
