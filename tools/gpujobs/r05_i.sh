# C2: more parts with one generator block per SM
mkdir -p gpurun_out/r05i
run() { echo "$1: $(FSMC_DRAW_BLOCKS_PER_SM=$2 FSMC_WIN_BLOCKS_PER_SM=$3 timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $4 $5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], d['roofline']['kernel_ms'])")"; }
{
run "p8 g1" 1 0 8
run "p10 g1" 1 0 10
run "p12 g1" 1 0 12
run "p16 g1" 1 0 16
run "p16 g2" 2 0 16
run "p12 g2" 2 0 12
run "p8 g1 W3003" 1 0 8 "--draw-window 3003"
run "p8 g1 W6006" 1 0 8 "--draw-window 6006"
run "p12 g1 W3003" 1 0 12 "--draw-window 3003"
run "p16 g1 W2002" 1 0 16 "--draw-window 2002"
run "p8 g1" 1 0 8
} > gpurun_out/r05i/sweep.txt 2>&1
cat gpurun_out/r05i/sweep.txt
