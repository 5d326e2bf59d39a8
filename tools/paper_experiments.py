"""Reproduce the paper's DRMH speed-up experiment on the B200 (§7.1):
N(0,1) target, N(x, 0.1^2) proposal, M = 100 tries, 10k samples per chain.
FSM (bundled, and the 4-way split body plain vs bundled) against the same-code
lock-step (vmap) baseline over a sweep of m; also the reference's efficiency
bound R(m) = E[max_j N] / E[N] from the measured per-sample step counts.

usage: python tools/paper_experiments.py [n] > profiles/rXX_paper_drmh.json
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
target = fm.standard_normal_target(1)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / 1e3


rows = []
for m in (1, 32, 1024, 16384, 65536):
    b = fm.drmh_kernel(100, 0.1)
    fsm_out, t_fsm = timed(lambda: fm.run_fsm_batched(b, target, fm.init_batch(b, target, m, 0), n,
                                                      step_variant="bundled", output="torch",
                                                      surplus=False))
    _, t_lock = timed(lambda: fm.run_standard_batched(b, target, fm.init_batch(b, target, m, 0), n,
                                                      output="torch"))
    N = fsm_out[1].iter_counts.to(torch.float64)
    burn = n // 5
    R = float(N[burn:].max(dim=1).values.mean() / N[burn:].mean())
    sb = fm.drmh_kernel(100, 0.1, split_body=True)
    _, lp = fm.run_fsm_batched(sb, target, fm.init_batch(sb, target, m, 0), n, step_variant="plain",
                               output="torch", surplus=False)
    _, lb = fm.run_fsm_batched(sb, target, fm.init_batch(sb, target, m, 0), n,
                               step_variant="bundled", output="torch", surplus=False)
    rows.append({"m": m, "n": n, "fsm_s": t_fsm, "lockstep_s": t_lock,
                 "speedup_vs_lockstep": t_lock / t_fsm, "R_m": R,
                 "fsm_samples_per_s": m * n / t_fsm,
                 "split_plain_over_bundled_ticks": lp.tick_count / lb.tick_count})
    print(json.dumps(rows[-1]), file=sys.stderr)
print(json.dumps({"experiment": "PAPER.md 7.1 DRMH: N(0,1), N(x,0.1) proposal, M=100",
                  "rows": rows}, indent=1))
