"""Symmetric delayed-rejection Metropolis-Hastings (drop-in for ``kernels/drmh.py``).

States INIT / PROPOSE / DONE, PROPOSE self-looping; each stage draws
y' = y + scale * eps (d counters), evaluates log p(y') and accepts with the
symmetric DR rule (``drmh.py:55-60``).  The blocks run on the device
(``Drmh`` in ``csrc/fsm_device.cuh``).
"""

from __future__ import annotations

from .. import _lib
from ..fsm import compose_single_loop
from ..lockstep import CostParams
from .base import KernelBundle, KernelError

__all__ = ["drmh_kernel"]


def drmh_kernel(max_tries: int, proposal_scale: float, split_body: bool = False) -> KernelBundle:
    """drmh.py:63-183 (the 4-way split body is not compiled on the device yet)."""
    if max_tries < 1:
        raise KernelError(f"max_tries must be >= 1, got {max_tries}")
    if not proposal_scale > 0:
        raise KernelError(f"proposal_scale must be positive, got {proposal_scale}")
    if split_body:
        raise KernelError("split_body=True (drmh.py:106-156) is not compiled on the device engine")
    machine = compose_single_loop(("INIT", "PROPOSE", "DONE"), family=_lib.DRMH)
    return KernelBundle(
        name="drmh", fsm=machine, family=_lib.DRMH, iter_states=(2,),
        default_costs=CostParams.for_fsm(machine, block_costs=(0.05, 1.0, 0.05)),
        max_tries=int(max_tries), proposal_scale=float(proposal_scale))
