#!/bin/bash
# On the GPU box: pipe ceilings (tools/peak_probe + cuBLAS DGEMM) and the fp64
# operation counts of the C2 step kernel, for the compute roofline.
mkdir -p gpurun_out
tools/peak_probe > gpurun_out/peaks.json; echo probe=$?
python - >> gpurun_out/peaks_dgemm.txt <<'PY'
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(2): a @ b
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5): a @ b
e1.record(); torch.cuda.synchronize()
print("dgemm_tflops", 5 * 2 * 8192**3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
PY
CMD="python bench.py --steps 1 --warmup 1 --n 200 --no-cpu --no-lockstep"
$CMD > gpurun_out/mix_plain.json 2>&1 && \
  timeout 900 ncu --clock-control none -k regex:fsm_run_kernel -s 1 -c 1 \
    --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --csv $CMD > gpurun_out/mix_ncu.csv 2> gpurun_out/mix_ncu.err
echo ncu=$?
