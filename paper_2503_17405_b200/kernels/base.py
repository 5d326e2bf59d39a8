"""Kernel bundles (drop-in for ``fsm_mcmc.kernels.base``).

A :class:`KernelBundle` names a compiled device kernel family and carries the
host metadata the drivers need: the machine shape, the loop states whose
executions make up N (``iter_states``), the default cost parameters and the
target requirements (``kernels/base.py:33-59``).  The ``fsmc_kernel``
descriptor is what crosses the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass

from .. import _lib
from ..fsm import FsmDefinition
from ..lockstep import CostParams

__all__ = ["KernelBundle", "KernelError"]


class KernelError(ValueError):
    """Invalid kernel construction or target/kernel mismatch (kernels/base.py:24-25)."""


@dataclass(frozen=True)
class KernelBundle:
    name: str
    fsm: FsmDefinition
    family: int
    iter_states: tuple
    default_costs: CostParams
    max_tries: int = 0
    proposal_scale: float = 0.0
    step_size: float = 0.0
    max_depth: int = 0
    divergence_threshold: float = 1000.0
    split_body: bool = False
    slice_width: float = 0.0
    max_expansions: int = 0

    def __post_init__(self):
        if not set(self.iter_states) <= self.fsm.loop_states:
            raise KernelError(f"{self.name}: iter_states {self.iter_states} must be loop states")

    def struct(self) -> _lib.Kernel:
        k = _lib.Kernel()
        k.family = self.family
        k.max_tries = self.max_tries
        k.proposal_scale = self.proposal_scale
        k.step_size = self.step_size
        k.max_depth = self.max_depth
        k.split_body = int(self.split_body)
        k.divergence_threshold = self.divergence_threshold
        k.slice_width = self.slice_width
        k.max_expansions = self.max_expansions
        return k

    def check_target(self, target) -> None:
        """kernels/base.py:55-59 with each kernel's ``requires``."""
        if self.family == _lib.ESS and target.gaussian_prior is None:
            raise KernelError(f"{self.name}: target lacks the Gaussian-prior decomposition")
        if self.family == _lib.NUTS and not target.has_gradient:
            raise KernelError(f"{self.name}: target lacks a gradient")
        if self.family == _lib.SLICE and target.dim != 1:   # slice_sampling.py:128-132
            raise KernelError(f"{self.name}: slice sampling here is univariate, target has dim "
                              f"{target.dim}")

    @property
    def loop_states(self) -> tuple:
        return tuple(sorted(self.fsm.loop_states))
