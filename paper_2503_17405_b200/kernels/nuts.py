"""Iterative No-U-Turn sampler (drop-in for ``kernels/nuts.py``).

Five states INIT / DOUBLE / INTEGRATE / CHECK / DONE (an outer doubling loop
around a leapfrog loop, ``fsm.py:348-388``); multinomial trajectory sampling
and progressive U-turn checkpoints (``nuts.py:48-61``), kept in HBM per chain.
"""

from __future__ import annotations

from .. import _lib
from ..fsm import compose_nested, compose_single_loop
from ..lockstep import CostParams
from .base import KernelBundle, KernelError

__all__ = ["nuts_kernel"]


def nuts_kernel(step_size: float, max_depth: int = 10,
                divergence_threshold: float = 1000.0) -> KernelBundle:
    """nuts.py:103-258"""
    if not step_size > 0:
        raise KernelError(f"step_size must be positive, got {step_size}")
    if max_depth < 1:
        raise KernelError(f"max_depth must be >= 1, got {max_depth}")
    if max_depth > 40:
        raise KernelError("max_depth above 40 is not supported")
    if not divergence_threshold > 0:
        raise KernelError("divergence_threshold must be positive")
    inner = compose_single_loop(("DOUBLE", "INTEGRATE", "CHECK"))
    machine = compose_nested(inner, ("INIT", "DONE"), family=_lib.NUTS)
    return KernelBundle(
        name="nuts", fsm=machine, family=_lib.NUTS, iter_states=(3,),
        default_costs=CostParams.for_fsm(machine, block_costs=(1.0, 0.05, 1.0, 0.1, 0.02)),
        step_size=float(step_size), max_depth=int(max_depth),
        divergence_threshold=float(divergence_threshold))
