"""The paper's section 7.2 experiment on the B200 (PAPER.md: elliptical slice
sampling of squared-exponential GP-regression hyperparameters, N(0, 1)
priors, n = 414 observations with 6 features, amortized log-pdf calls).
The UCI real-estate data is not available offline: a synthetic dataset of
the same shape is drawn from the GP model itself (make_synthetic_gp_dataset,
the reference's generator).  Every log-pdf call is a 414 x 414 Cholesky, done
for all requesting chains at once (dense.GPHyperEvaluator).

FSM (amortized: one batched evaluation per round) against the same-code
lock-step baseline (fsmc_advance_lockstep: a barrier at every sample, the
whole batch evaluated every round, as vmap with while loops), over m.
Reports wall times, their ratio, rounds (= batched log-pdf calls), mean
iterations per sample (FSM: mean over chains; lock-step: max over chains,
which the paper plots growing from 6 to 18) and R(m).

usage: python tools/paper_gp_experiment.py [n_samples] [m ...] > profiles/rXX_paper_gp.json
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ms = [int(v) for v in sys.argv[2:]] or [1, 128, 1024]
X, y = fm.make_synthetic_gp_dataset(414, 6)
target = fm.gp_hyperparameter_target(X, y)
x0 = torch.tensor([0.3, 1.0, 1.0], dtype=torch.float64)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / 1e3


b = fm.elliptical_kernel()
timed(lambda: fm.run_fsm_batched(b, target, fm.init_batch(b, target, 8, 99, x0=x0), 5,
                                 step_variant="amortized", output="torch"))   # warm-up
rows = []
for m in ms:
    (s_f, l_f), t_f = timed(lambda: fm.run_fsm_batched(b, target, fm.init_batch(b, target, m, 0, x0=x0),
                                                       n, step_variant="amortized", output="torch",
                                                       surplus=False))
    (s_l, l_l), t_l = timed(lambda: fm.run_standard_batched(b, target,
                                                            fm.init_batch(b, target, m, 0, x0=x0), n,
                                                            output="torch"))
    N = l_f.iter_counts.to(torch.float64)            # SHRINK executions per sample
    burn = n // 5
    its_fsm = float(N[burn:].mean()) + 1.0           # + the INIT evaluation
    its_lock = float(N[burn:].max(dim=1).values.mean()) + 1.0
    ess = fm.effective_sample_size(s_f[n // 10:]).pooled if n >= 100 else None
    rows.append({"m": m, "n": n, "fsm_s": t_f, "lockstep_s": t_l, "speedup_vs_lockstep": t_l / t_f,
                 "fsm_rounds": l_f.extras["rounds"], "lockstep_rounds": l_l.extras["rounds"],
                 "fsm_evaluations": l_f.extras["evaluations"],
                 "lockstep_evaluations": l_l.extras["evaluations"],
                 "evals_per_sample_fsm_mean": its_fsm, "evals_per_sample_lockstep": its_lock,
                 "R_m": its_lock / its_fsm, "fsm_samples_per_s": m * n / t_f,
                 "fsm_ess_per_s": None if ess is None else ess / t_f})
    print(json.dumps(rows[-1]), file=sys.stderr)
print(json.dumps({"experiment": "PAPER.md 7.2: ESS on GP-regression hyperparameters, n=414 x 6 "
                                "(synthetic, same shape), amortized, batched fp64 Cholesky per round",
                  "rows": rows}, indent=1))
