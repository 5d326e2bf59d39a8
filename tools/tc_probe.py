"""Time the fused tcgen05 logistic-regression kernel alone (CUDA events)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_17405_b200.dense import LogisticRegressionEvaluator  # noqa: E402
from paper_2503_17405_b200.targets import logistic_regression_data  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16-tc"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
X, y = logistic_regression_data(100_000, 256, seed=0)
ev = LogisticRegressionEvaluator(X, y, precision=prec)
th = torch.randn(k, 256, dtype=torch.float64, device="cuda") * 0.1
lp = torch.empty(k, dtype=torch.float64, device="cuda")
g = torch.empty((k, 256), dtype=torch.float64, device="cuda")
ev(th, lp, g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ev(th, lp, g)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
flops = 4.0 * 100_000 * 256 * k
print(f"{prec} k={k}: {ms:.3f} ms/eval-round, {flops / ms / 1e9:.1f} TFLOP/s")
