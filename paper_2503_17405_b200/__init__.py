"""B200-native multi-chain FSM MCMC engine (arXiv 2503.17405).

Drop-in for the reference package ``fsm_mcmc``'s multi-chain sampling path:
the same kernel builders, batch drivers, executors and plugin names, backed
by hand-written sm_100a CUDA kernels (``libfsmc.so``, C ABI in
``include/fsmc.h``).  There is no CPU fallback.
"""

import os as _os

# The windowed DRMH run drives up to 16 chain-part streams plus a
# device-to-host egress stream.  With CUDA's default of 8 hardware work
# queues per device, streams share queues and an egress copy stalls the
# kernels queued behind it on an unrelated part (measured on B200: C2 with
# host output 220 ms -> 176 ms per step at 32 queues).  Read once, when the
# process creates its CUDA context; an explicit setting is kept.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .fsm import (BlockFailure, FsmDefinition, FsmError, SharedComputation, StepOutcome,
                  amortized_step, bundled_step, compose_nested, compose_sequential,
                  compose_single_loop, step)
from .kernels import KERNEL_BUILDERS, KernelBundle, KernelError, drmh_kernel, elliptical_kernel, \
    nuts_kernel, slice_kernel
from .lockstep import (ChainBatch, CostLedger, CostParams, KernelRunError, TickBudgetExceeded,
                       collect_samples, init_batch, measure_block_costs, run_fsm_batched,
                       run_standard_batched)
from .prng import RngKey, key, normal, normal_vec, split, uniform, uniform_block
from .targets import (GaussianPriorDecomposition, TargetError, TargetModel, batched_target,
                      conjugate_target,
                      correlated_mog_target, equicorrelated_covariance,
                      box_target, equicorrelated_gaussian_target, funnel_target, gaussian_target,
                      gp_classification_target, gp_hyperparameter_target,
                      load_gp_dataset_csv, make_synthetic_gp_dataset, save_gp_dataset_csv,
                      standard_normal_target)
from .analysis import EssSummary, effective_sample_size, rhat

__version__ = "0.1.0"
