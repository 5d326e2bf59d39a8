# C2 under bounded generators: generator variants, generator grid, slots
mkdir -p gpurun_out/r05y
bash tools/ab.sh "--steps 8 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/u2/libfsmc.so variants/u8/libfsmc.so variants/minb2/libfsmc.so variants/tail1/libfsmc.so paper_2503_17405_b200/libfsmc.so > gpurun_out/r05y/ab.txt 2>&1
cat gpurun_out/r05y/ab.txt
for cfg in "1 0" "3 0" "2 1" "2 2" "2 4" "1 1" "4 0"; do set -- $cfg
  FSMC_GEN_SLOTS=$1 FSMC_DRAW_BLOCKS_PER_SM=$2 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e > gpurun_out/r05y/r.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r05y/r.json').read().strip().splitlines()[-1]); print('p8 slots$1 g$2', '%.4g'%d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done
