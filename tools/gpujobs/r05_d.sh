# C2: how much the part overlap buys (draw_parts 1/2/4/8)
mkdir -p gpurun_out/r05d
for P in 1 2 4 8; do echo "parts $P: $(timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-lockstep --no-e2e --draw-parts $P 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], d['roofline']['kernel_ms'])")"; done > gpurun_out/r05d/parts.txt 2>&1
cat gpurun_out/r05d/parts.txt
