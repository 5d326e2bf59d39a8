"""Small invocations of every kernel family for compute-sanitizer (one tool per
gpurun call: memcheck, racecheck, synccheck).  Each step is checked against
its own expectation so a silent failure under the tool still shows.

  compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2503_17405_b200 as fm
    from paper_2503_17405_b200.dense import LogisticRegressionEvaluator
    from paper_2503_17405_b200.targets import logistic_regression_data

    mog = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
    dr = fm.drmh_kernel(20, 0.3)
    a, la = fm.run_fsm_batched(dr, mog, fm.init_batch(dr, mog, 96, 1), 12, step_variant="bundled")
    b, lb = fm.run_fsm_batched(dr, mog, fm.init_batch(dr, mog, 96, 1), 12, step_variant="bundled",
                               draw_window=220, draw_parts=2)
    assert np.array_equal(a, b), "windowed run differs"
    c, lc = fm.run_standard_batched(dr, mog, fm.init_batch(dr, mog, 96, 1), 12)
    assert np.array_equal(a, c), "lock-step differs"
    f32, _ = fm.run_fsm_batched(dr, mog, fm.init_batch(dr, mog, 96, 1), 12, step_variant="bundled",
                                precision="fp32")
    assert np.isfinite(f32).all()
    print("drmh ok")

    nu = fm.nuts_kernel(0.05, 6)
    eq = fm.equicorrelated_gaussian_target(100, 0.99)
    s, _ = fm.run_fsm_batched(nu, eq, fm.init_batch(nu, eq, 8, 2), 3, step_variant="bundled")
    s2, _ = fm.run_standard_batched(nu, eq, fm.init_batch(nu, eq, 8, 2), 3)
    assert np.array_equal(s, s2), "nuts lock-step differs"
    print("nuts ok")

    es = fm.elliptical_kernel()
    gp = fm.gp_classification_target(128)
    e1, l1 = fm.run_fsm_batched(es, gp, fm.init_batch(es, gp, 16, 3), 3, step_variant="amortized")
    e2, l2 = fm.run_fsm_batched(es, gp, fm.init_batch(es, gp, 16, 3), 3, step_variant="amortized",
                                prior_transform="dmma", prior_parts=2)
    assert np.array_equal(l1.iter_counts, l2.iter_counts), "dmma prior changes step counts"
    print("ess ok")

    X, y = logistic_regression_data(256, 256, seed=1)
    ev = LogisticRegressionEvaluator(X, y, precision="fp16-tc")
    th = torch.randn(130, 256, dtype=torch.float64, device="cuda") * 0.2
    lp = torch.empty(130, dtype=torch.float64, device="cuda")
    g = torch.empty((130, 256), dtype=torch.float64, device="cuda")
    ev(th, lp, g)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(lp).all()) and bool(torch.isfinite(g).all())
    print("logreg_tc ok")

    ess = fm.effective_sample_size(a, burn=0)
    assert np.isfinite(ess.pooled)
    print("diagnostics ok")


if __name__ == "__main__":
    main()
    print("sanitize probe done")
