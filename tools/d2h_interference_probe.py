"""Does a concurrent device-to-host copy stream slow the C2 kernels?  The run
(output="torch", 12 parts) alone, then with a side stream copying an unrelated
1 GB buffer to pinned memory over and over during it."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402

b = fm.drmh_kernel(100, 0.1)
t = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
m, n = 65536, 1000
src = torch.randn(1 << 27, dtype=torch.float64, device="cuda")      # 1 GB
dst = torch.empty(1 << 27, dtype=torch.float64, pin_memory=True)
side = torch.cuda.Stream()
for copies in (0, 0, 8, 8, 16, 0):
    batch = fm.init_batch(b, t, m, 7)
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        for _ in range(copies):
            dst.copy_(src, non_blocking=True)
    tim = {}
    t0 = time.perf_counter()
    s, led = fm.run_fsm_batched(b, t, batch, n, step_variant="bundled", output="torch", surplus=False,
                                draw_window=4070, draw_parts=int(sys.argv[1]) if len(sys.argv) > 1 else 12,
                                _timing=tim)
    torch.cuda.synchronize()
    print(f"{copies} GB copied alongside: run kernels {tim['run_kernel_ms']:.1f} ms, "
          f"wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del s, led
