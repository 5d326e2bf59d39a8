"""Where the bench's end-to-end step goes (C2 by default): init_batch,
run_fsm_batched, effective_sample_size, each timed with CUDA events."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2503_17405_b200 as fm  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
bundle, target = bench.make_workload(cfg, fm)
m, n = cfg["m"], cfg["n"]
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch = fm.init_batch(bundle, target, m, 500 + it)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    smp, _ = fm.run_fsm_batched(bundle, target, batch, n, step_variant=cfg["variant"], output="torch",
                                surplus=False, draw_window=cfg.get("draw_window", 0),
                                draw_parts=cfg.get("draw_parts", 1),
                                prior_transform=cfg.get("prior_transform"))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ess = fm.effective_sample_size(smp, burn=n // 10).pooled
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"init {1e3 * (t1 - t0):.1f} ms  run {1e3 * (t2 - t1):.1f} ms  ess {1e3 * (t3 - t2):.1f} ms"
          f"  (pooled ESS {ess:.0f})")
