"""Elliptical slice sampling (drop-in for ``kernels/elliptical.py``).

States INIT / SHRINK / DONE; the residual log-density is the shared
computation, requested by INIT and SHRINK and evaluated once per request
between block and transition (``elliptical.py:61-62, 210-211``).
"""

from __future__ import annotations

from .. import _lib
from ..fsm import SharedComputation, compose_single_loop
from ..lockstep import CostParams
from .base import KernelBundle

__all__ = ["elliptical_kernel"]


def elliptical_kernel() -> KernelBundle:
    """elliptical.py:65-142"""
    shared = SharedComputation(sites={1: 1, 2: 1}, label="residual log-density")
    machine = compose_single_loop(("INIT", "SHRINK", "DONE"), shared=shared, family=_lib.ESS)
    return KernelBundle(
        name="elliptical", fsm=machine, family=_lib.ESS, iter_states=(2,),
        default_costs=CostParams.for_fsm(machine, block_costs=(0.02, 0.02, 0.01),
                                         shared_cost=1.0))
