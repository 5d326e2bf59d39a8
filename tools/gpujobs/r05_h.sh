# C2 (4 parts): generator / window-kernel blocks per SM
mkdir -p gpurun_out/r05h
run() { echo "$1: $(FSMC_DRAW_BLOCKS_PER_SM=$2 FSMC_WIN_BLOCKS_PER_SM=$3 timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], d['roofline']['kernel_ms'])")"; }
{
run "p4 g0 w0" 0 0 4
run "p4 g2 w2" 2 2 4
run "p4 g2 w0" 2 0 4
run "p4 g0 w2" 0 2 4
run "p4 g3 w2" 3 2 4
run "p4 g2 w1" 2 1 4
run "p4 g1 w1" 1 1 4
run "p8 g2 w2" 2 2 8
run "p8 g1 w1" 1 1 8
run "p2 g2 w2" 2 2 2
run "p4 g4 w4" 4 4 4
run "p4 g0 w0" 0 0 4
} > gpurun_out/r05h/sweep.txt 2>&1
cat gpurun_out/r05h/sweep.txt
