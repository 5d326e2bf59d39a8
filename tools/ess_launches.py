"""One C4-sized effective_sample_size call after a warm-up (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402
n, m, d = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (200, 8192, 1024)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((n, m, d), dtype=torch.float64, device="cuda", generator=g)
for i in range(1, n):          # AR(1) rows, rho = 0.99: Geyer needs every lag
    x[i].mul_(0.141).add_(x[i - 1], alpha=0.99)
for _ in range(2):
    fm.effective_sample_size(x, burn=n // 10)
torch.cuda.synchronize()
