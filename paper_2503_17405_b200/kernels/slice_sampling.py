"""Univariate slice sampling with stepping-out and shrinkage (drop-in for
``kernels/slice_sampling.py``).

Five states from the sequential composition of two single-loop machines
(``fsm.py:307-345``): INIT-E draws the level and the initial bracket and
evaluates both ends, EXPAND steps one end out per execution (left first),
INIT-S is empty, SHRINK proposes inside the bracket until a point lands above
the level, DONE moves the chain.  The blocks run on the device (``Slice`` in
``csrc/fsm_device.cuh``); hitting the expansion cap is counted, not an error.
"""

from __future__ import annotations

from .. import _lib
from ..fsm import compose_sequential, compose_single_loop
from ..lockstep import CostParams
from .base import KernelBundle, KernelError

__all__ = ["slice_kernel"]


def slice_kernel(initial_width: float, max_expansions: int = 32) -> KernelBundle:
    """slice_sampling.py:50-156: stepping-out/shrinkage for one-dimensional targets."""
    if not initial_width > 0:
        raise KernelError(f"initial_width must be positive, got {initial_width}")
    if max_expansions < 0:
        raise KernelError(f"max_expansions must be >= 0, got {max_expansions}")
    machine = compose_sequential(compose_single_loop(("INIT-E", "EXPAND", "INIT-S")),
                                 compose_single_loop(("INIT-S", "SHRINK", "DONE")),
                                 family=_lib.SLICE)
    return KernelBundle(
        name="slice", fsm=machine, family=_lib.SLICE, iter_states=(2, 4),
        default_costs=CostParams.for_fsm(machine), slice_width=float(initial_width),
        max_expansions=int(max_expansions))
