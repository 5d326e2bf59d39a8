# round 2: progress-check interval (e2e tail of the streamed rows)
mkdir -p gpurun_out/r04t
for L in paper_2503_17405_b200/libfsmc.so variants/k4/libfsmc.so paper_2503_17405_b200/libfsmc.so; do
  FSMC_LIB=$(realpath $L) timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-lockstep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$L', '%.4g'%d['value'], 'kernel %.1f'%d['roofline']['kernel_ms'], 'e2e %.4g'%d['e2e']['value'], d['e2e']['ms'])"
done > gpurun_out/r04t/ab.txt 2>&1; cat gpurun_out/r04t/ab.txt
