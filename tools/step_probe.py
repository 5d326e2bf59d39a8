import sys, time, torch
sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm
from paper_2503_17405_b200 import lockstep as L
b = fm.drmh_kernel(100, 0.1); t = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
m, n = 65536, 1000
def step(seed):
    t0 = time.perf_counter()
    batch = fm.init_batch(b, t, m, seed)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    tim = {}
    s, led = fm.run_fsm_batched(b, t, batch, n, step_variant="bundled", output="torch", surplus=False, _timing=tim)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3, tim["run_kernel_ms"]
for i in range(6):
    print([round(x, 2) for x in step(i)])
