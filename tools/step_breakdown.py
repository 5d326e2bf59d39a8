"""Where a C2 bench step's wall time goes beyond the step kernel (GPU box)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_17405_b200 as fm

b = fm.drmh_kernel(100, 0.1)
t = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
m, n = 65536, 1000
win = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    batch = fm.init_batch(b, t, m, it)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    timing = {}
    s, led = fm.run_fsm_batched(b, t, batch, n, step_variant="bundled", output="torch", surplus=False,
                                draw_window=win, _timing=timing)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"init {1e3*(t1-t0):7.2f} ms  run {1e3*(t2-t1):7.2f} ms  kernel {timing['run_kernel_ms']:7.2f} ms  "
          f"reserved {torch.cuda.memory_reserved()/2**30:.1f} GiB")
