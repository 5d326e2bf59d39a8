# round 2: C2 window-size sweep above 4096 draws
mkdir -p gpurun_out/r04q
for pw in "4 4070" "4 6000" "4 8180" "4 12000" "4 16000" "3 8180" "8 8180"; do set -- $pw
  V=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-lockstep --draw-parts $1 --draw-window $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f'{d[\"value\"]:.4g} kernel {d[\"roofline\"][\"kernel_ms\"]:.1f} ms')")
  echo "parts $1 window $2: $V"
done > gpurun_out/r04q/sweep.txt 2>&1; cat gpurun_out/r04q/sweep.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "windowed" > gpurun_out/r04q/tests.log 2>&1; tail -1 gpurun_out/r04q/tests.log
