# pipelined windows (draw_parts=0): parity, then generator/window blocks-per-SM sweep
mkdir -p gpurun_out/r05e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed" > gpurun_out/r05e/parity.log 2>&1; tail -3 gpurun_out/r05e/parity.log
run() { echo "$1: $(FSMC_DRAW_BLOCKS_PER_SM=$2 FSMC_WIN_BLOCKS_PER_SM=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], d['roofline']['kernel_ms'])")"; }
{
run "parts4 default" 0 0 4
run "pipe default" 0 0 0
run "pipe g1 w3" 1 3 0
run "pipe g2 w2" 2 2 0
run "pipe g1 w2" 1 2 0
run "pipe g2 w1" 2 1 0
run "pipe g3 w1" 3 1 0
run "pipe g2 w3" 2 3 0
run "parts4 g2 w2" 2 2 4
} > gpurun_out/r05e/sweep.txt 2>&1
cat gpurun_out/r05e/sweep.txt
