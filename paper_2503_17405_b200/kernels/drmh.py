"""Symmetric delayed-rejection Metropolis-Hastings (drop-in for ``kernels/drmh.py``).

States INIT / PROPOSE / DONE, PROPOSE self-looping; each stage draws
y' = y + scale * eps (d counters), evaluates log p(y') and accepts with the
symmetric DR rule (``drmh.py:55-60``).  The blocks run on the device
(``Drmh`` in ``csrc/fsm_device.cuh``).
"""

from __future__ import annotations

from .. import _lib
from ..fsm import FsmDefinition, compose_single_loop
from ..lockstep import CostParams
from .base import KernelBundle, KernelError

__all__ = ["drmh_kernel"]


def drmh_kernel(max_tries: int, proposal_scale: float, split_body: bool = False) -> KernelBundle:
    """drmh.py:63-183.  ``split_body=True`` unrolls PROPOSE into PROP-DRAW /
    PROP-EVAL / PROP-TEST / PROP-APPLY (drmh.py:106-156), the machine of the
    paper's step-bundling experiment; same draws, same samples."""
    if max_tries < 1:
        raise KernelError(f"max_tries must be >= 1, got {max_tries}")
    if not proposal_scale > 0:
        raise KernelError(f"proposal_scale must be positive, got {proposal_scale}")
    if split_body:
        machine = FsmDefinition(
            labels=("INIT", "PROP-DRAW", "PROP-EVAL", "PROP-TEST", "PROP-APPLY", "DONE"),
            edges=frozenset({(1, 2), (1, 6), (2, 3), (3, 4), (4, 5), (5, 2), (5, 6), (6, 1)}),
            loop_states=frozenset({2, 3, 4, 5}), family=_lib.DRMH)
        costs = (0.05, 1.0, 1.0, 1.0, 1.0, 0.05)
    else:
        machine = compose_single_loop(("INIT", "PROPOSE", "DONE"), family=_lib.DRMH)
        costs = (0.05, 1.0, 0.05)
    return KernelBundle(
        name="drmh-split" if split_body else "drmh", fsm=machine, family=_lib.DRMH,
        iter_states=(2,), default_costs=CostParams.for_fsm(machine, block_costs=costs),
        max_tries=int(max_tries), proposal_scale=float(proposal_scale), split_body=bool(split_body))
