"""C2 step breakdown for the windowed-run modes: host time of init_batch and
run_fsm_batched, the run's event-timed kernel span, per draw_parts setting.
usage: python tools/pipe_probe.py PARTS [PARTS ...]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402

b = fm.drmh_kernel(100, 0.1)
t = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
m, n = 65536, 1000
for parts in [int(v) for v in sys.argv[1:]]:
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch = fm.init_batch(b, t, m, i)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        tim = {}
        s, led = fm.run_fsm_batched(b, t, batch, n, step_variant="bundled", output="torch",
                                    surplus=False, draw_window=4070, draw_parts=parts, _timing=tim)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"parts {parts}: init {1e3 * (t1 - t0):.1f} ms, run host {1e3 * (t2 - t1):.1f} ms "
              f"(+sync {1e3 * (t3 - t2):.1f}), run kernels {tim['run_kernel_ms']:.1f} ms", flush=True)
        del s, led
