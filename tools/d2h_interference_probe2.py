"""Egress-pattern copies alongside the C2 run: bursts of pitched 2D copies
(part column blocks of ~27 sample rows) into pinned memory, issued from the
host every few ms while the run proceeds on other streams, vs one big copy."""
import ctypes
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402
from paper_2503_17405_b200 import _lib  # noqa: E402

b = fm.drmh_kernel(100, 0.1)
t = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
m, n, d = 65536, 1000, 10
src = torch.randn(n, m, d, dtype=torch.float64, device="cuda")
dst = torch.empty(n, m, d, dtype=torch.float64, pin_memory=True)
side = torch.cuda.Stream()
lib = _lib.lib()
pitch = m * d * 8


def feeder(parts, rows_per_burst, period_s, stop):
    r = 0
    while not stop.is_set() and r < n:
        for h in range(parts):
            lo, hi = m * h // parts, m * (h + 1) // parts
            nr = min(rows_per_burst, n - r)
            if parts == 0:
                break
            lib.fsmc_copy_to_host_2d(dst.data_ptr() + r * pitch + lo * d * 8,
                                     src.data_ptr() + r * pitch + lo * d * 8, pitch, (hi - lo) * d * 8, nr,
                                     ctypes.c_void_p(side.cuda_stream))
        r += rows_per_burst
        time.sleep(period_s)


for parts in (0, 12, 1, 12):
    batch = fm.init_batch(b, t, m, 7)
    torch.cuda.synchronize()
    stop = threading.Event()
    th = threading.Thread(target=feeder, args=(parts, 27, 0.0044, stop))
    tim = {}
    t0 = time.perf_counter()
    th.start()
    s, led = fm.run_fsm_batched(b, t, batch, n, step_variant="bundled", output="torch", surplus=False,
                                draw_window=4070, draw_parts=12, _timing=tim)
    torch.cuda.synchronize()
    stop.set()
    th.join()
    torch.cuda.synchronize()
    print(f"feeder parts {parts}: run kernels {tim['run_kernel_ms']:.1f} ms, wall {1e3 * (time.perf_counter() - t0):.1f} ms",
          flush=True)
    del s, led
