"""NUTS on the GP-hyperparameter target above the per-chain plugin's 56
observations (deferred init + batched-evaluation rounds, the gradient by
fsmc_gp_lml_grad).  Run under `ncu --metrics gpu__time_duration.sum --csv`
to list every kernel the run launches (no cuSOLVER / cuBLAS kernel expected).
usage: python tools/gp_nuts_launches.py [n_obs]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_17405_b200 as fm  # noqa: E402

n_obs = int(sys.argv[1]) if len(sys.argv) > 1 else 90
X, y = fm.make_synthetic_gp_dataset(n_obs, 6)
t = fm.gp_hyperparameter_target(X, y)
b = fm.nuts_kernel(0.05, 6)
s, led = fm.run_fsm_batched(b, t, fm.init_batch(b, t, 64, 2, x0=np.array([0.3, 1.0, 1.0])), 10,
                            step_variant="bundled", surplus=False)
torch.cuda.synchronize()
print(f"NUTS on the GP target, n_obs={n_obs}: rounds {led.extras['rounds']}, samples {np.asarray(s).shape}")
