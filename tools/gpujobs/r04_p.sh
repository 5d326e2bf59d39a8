# round 2: C2 window-kernel occupancy variants and draw-part / window-size sweep
mkdir -p gpurun_out/r04p
bash tools/ab.sh "--steps 5 --warmup 3 --no-e2e" paper_2503_17405_b200/libfsmc.so variants/w5/libfsmc.so variants/w6/libfsmc.so > gpurun_out/r04p/ab_occ.txt 2>&1; cat gpurun_out/r04p/ab_occ.txt
for pw in "4 4070" "6 4070" "8 4070" "4 3000" "3 4070" "2 4070"; do set -- $pw
  V=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-lockstep --draw-parts $1 --draw-window $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f'{d[\"value\"]:.4g} kernel {d[\"roofline\"][\"kernel_ms\"]:.1f} ms')")
  echo "parts $1 window $2: $V"
done > gpurun_out/r04p/sweep.txt 2>&1; cat gpurun_out/r04p/sweep.txt
