"""C2 e2e composition per chain-part count: run_fsm_batched wall time with
output="numpy" (rows streamed to pinned memory during the run) against
output="torch", and the run's event-timed kernel span.
usage: python tools/e2e_parts_probe.py PARTS [PARTS ...]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402

b = fm.drmh_kernel(100, 0.1)
t = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
m, n = 65536, 1000
for parts in [int(v) for v in sys.argv[1:]]:
    for output in ("torch", "numpy", "numpy", "numpy"):
        batch = fm.init_batch(b, t, m, 7)
        torch.cuda.synchronize()
        tim = {}
        t0 = time.perf_counter()
        s, led = fm.run_fsm_batched(b, t, batch, n, step_variant="bundled", output=output,
                                    surplus=False, draw_window=4070, draw_parts=parts, _timing=tim)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"parts {parts:2d} {output}: wall {1e3 * dt:.1f} ms, run kernels {tim['run_kernel_ms']:.1f} ms",
              flush=True)
        del s, led
