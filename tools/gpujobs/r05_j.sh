# C2: window size at 12 / 16 parts
mkdir -p gpurun_out/r05j
run() { echo "$1: $(FSMC_DRAW_BLOCKS_PER_SM=$2 FSMC_WIN_BLOCKS_PER_SM=$3 timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $4 $5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], d['roofline']['kernel_ms'])")"; }
{
run "p12 g1 W4070" 1 0 12
run "p12 g1 W5005" 1 0 12 "--draw-window 5005"
run "p12 g1 W6006" 1 0 12 "--draw-window 6006"
run "p12 g1 W8008" 1 0 12 "--draw-window 8008"
run "p16 g1 W5005" 1 0 16 "--draw-window 5005"
run "p16 g1 W6006" 1 0 16 "--draw-window 6006"
run "p16 g1 W8008" 1 0 16 "--draw-window 8008"
run "p14 g1 W6006" 1 0 14 "--draw-window 6006"
run "p12 g0 W6006" 0 0 12 "--draw-window 6006"
run "p12 g1 W4070" 1 0 12
} > gpurun_out/r05j/sweep.txt 2>&1
cat gpurun_out/r05j/sweep.txt
