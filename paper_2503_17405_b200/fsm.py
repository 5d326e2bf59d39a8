"""State-machine metadata and the single-chain executors (drop-in for ``fsm_mcmc.fsm``).

On the device a kernel's blocks are compiled code (``csrc/fsm_device.cuh``),
so an :class:`FsmDefinition` here carries the machine's *shape*: state labels,
the declared edge set, loop states and the shared-computation sites.  The
same validation rules as the reference apply (``fsm.py:117-149``): states
1..K, the final state's only edge wraps to 1, every state reachable.

``step`` / ``bundled_step`` / ``amortized_step`` advance ONE chain of a
device :class:`~paper_2503_17405_b200.lockstep.ChainBatch` by one executor
call (``fsm.py:182-273``); they exist for tests and tooling.  The hot path
is ``run_fsm_batched``, which runs every chain for many ticks in one launch.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, NamedTuple

__all__ = [
    "FsmError", "BlockFailure", "FsmDefinition", "SharedComputation", "StepOutcome",
    "ChainView", "step", "bundled_step", "amortized_step", "default_bundled_order",
    "validate_bundled_order", "compose_single_loop", "compose_sequential", "compose_nested",
    "topology_as_dict", "topology_as_graphviz",
]


class FsmError(ValueError):
    """Invalid state-machine structure or usage (fsm.py:56-57)."""


class BlockFailure(RuntimeError):
    """A block produced a NaN or +inf log-density; carries the state label (fsm.py:60-65)."""

    def __init__(self, label: str, message: str):
        super().__init__(f"[{label}] {message}")
        self.label = label


@dataclass(frozen=True)
class SharedComputation:
    """Where a machine's expensive shared function would be inlined (fsm.py:86-97).

    ``sites`` maps state -> call sites; the device evaluates it once per
    request between block and transition, exactly the reference protocol.
    """

    sites: dict
    label: str = "shared"


@dataclass(frozen=True)
class FsmDefinition:
    """A machine's shape: K state labels, declared edges, loop states."""

    labels: tuple
    edges: frozenset
    loop_states: frozenset = frozenset()
    shared: SharedComputation | None = None
    family: int = 0

    def __post_init__(self):
        K = len(self.labels)
        if K < 1:
            raise FsmError("a state machine needs at least one state")
        for a, b in self.edges:
            if not (1 <= a <= K and 1 <= b <= K):
                raise FsmError(f"edge ({a}, {b}) outside states 1..{K}")
        if {e for e in self.edges if e[0] == K} != {(K, 1)}:
            raise FsmError(f"final state must have exactly the wrap-around edge ({K}, 1)")
        if not set(self.loop_states) <= set(range(1, K + 1)):
            raise FsmError("loop_states outside 1..K")
        reach, todo = {1}, [1]
        while todo:
            a = todo.pop()
            for s, t in self.edges:
                if s == a and t not in reach:
                    reach.add(t)
                    todo.append(t)
        if reach != set(range(1, K + 1)):
            raise FsmError(f"states {sorted(set(range(1, K + 1)) - reach)} unreachable")

    @property
    def n_states(self) -> int:
        return len(self.labels)

    @property
    def initial(self) -> int:
        return 1

    @property
    def final(self) -> int:
        return len(self.labels)


class StepOutcome(NamedTuple):
    """Result of one executor call on one chain (fsm.py:164-171)."""

    state: int
    locals: Any
    is_sample: bool
    do_computation: bool
    executed: tuple


def default_bundled_order(fsm: FsmDefinition) -> tuple:
    """Final-first cyclic order (K, 1, ..., K-1) (fsm.py:198-208)."""
    K = fsm.n_states
    return (K, *range(1, K))


def validate_bundled_order(fsm: FsmDefinition, order) -> None:
    """Reject orders that would let a chain pass the final state unflagged (fsm.py:211-227)."""
    K = fsm.n_states
    order = tuple(order)
    if sorted(order) != list(range(1, K + 1)):
        raise FsmError(f"order {order} is not a permutation of 1..{K}")
    pos = {s: i for i, s in enumerate(order)}
    for a, b in fsm.edges:
        if b == K and a != K and pos[K] > pos[a]:
            raise FsmError(f"order {order} can swallow samples: edge {a}->{K} fires the final "
                           f"block after conditional {a} in the same call")


def compose_single_loop(labels=("INIT", "BODY", "DONE"), shared=None, family=0) -> FsmDefinition:
    """Three states, one while loop (fsm.py:281-304)."""
    return FsmDefinition(labels=tuple(labels),
                         edges=frozenset({(1, 2), (1, 3), (2, 2), (2, 3), (3, 1)}),
                         loop_states=frozenset({2}), shared=shared, family=family)


def compose_sequential(f1: FsmDefinition, f2: FsmDefinition, family: int = 0) -> FsmDefinition:
    """Two single-loop machines back to back -> five states (fsm.py:307-345)."""
    if f1.n_states != 3 or f2.n_states != 3:
        raise FsmError("sequential composition expects two single-loop machines")
    if f1.shared is not None or f2.shared is not None:
        raise FsmError("sequential composition of shared computations is not supported")
    return FsmDefinition(labels=(*f1.labels, f2.labels[1], f2.labels[2]),
                         edges=frozenset({(1, 2), (1, 3), (2, 2), (2, 3), (3, 4), (3, 5),
                                          (4, 4), (4, 5), (5, 1)}),
                         loop_states=frozenset({2, 4}), family=family)


def compose_nested(inner: FsmDefinition, labels=("INIT", "DONE"), family=0) -> FsmDefinition:
    """An outer loop around a single-loop body -> five states (fsm.py:348-388)."""
    if inner.n_states != 3:
        raise FsmError("nested composition expects a single-loop inner machine")
    return FsmDefinition(labels=(labels[0], *inner.labels, labels[1]),
                         edges=frozenset({(1, 2), (1, 5), (2, 3), (2, 4), (3, 3), (3, 4),
                                          (4, 2), (4, 5), (5, 1)}),
                         loop_states=frozenset({2, 3, 4}), shared=inner.shared, family=family)


def topology_as_dict(fsm: FsmDefinition) -> dict:
    return {"states": [{"id": i + 1, "label": lab} for i, lab in enumerate(fsm.labels)],
            "initial": 1, "final": fsm.final, "loop_states": sorted(fsm.loop_states),
            "edges": sorted([a, b] for a, b in fsm.edges)}


def topology_as_graphviz(fsm: FsmDefinition) -> str:
    out = ["digraph fsm {", "  rankdir=LR;"]
    for i, lab in enumerate(fsm.labels, start=1):
        out.append(f'  s{i} [label="{lab}", shape={"doublecircle" if i == fsm.final else "circle"}];')
    out += [f"  s{a} -> s{b};" for a, b in sorted(fsm.edges)]
    out.append("}")
    return "\n".join(out)


# ------------------------------------------------------------- single chain
@dataclass
class ChainView:
    """One chain of a device batch: what the reference calls the chain's Locals."""

    batch: Any
    index: int
    extra: dict = field(default_factory=dict)

    @property
    def x(self):
        return self.batch.chain_position(self.index)

    @property
    def rng(self):
        return self.batch.chain_key(self.index)


def _single(fsm: FsmDefinition, k: int, z: ChainView, variant: int, order=None) -> StepOutcome:
    if not isinstance(z, ChainView):
        raise FsmError("device executors step a ChainView (batch.chain(j)); "
                       "Python-callable blocks are not executable on the device")
    if not 1 <= k <= fsm.n_states:
        raise FsmError(f"state {k} outside 1..{fsm.n_states}")
    return z.batch._step_one(z.index, k, variant, order)


def step(fsm: FsmDefinition, k: int, z) -> StepOutcome:
    """One block + shared refresh + transition (fsm.py:182-195)."""
    return _single(fsm, k, z, 0)


def bundled_step(fsm: FsmDefinition, k: int, z, order=None) -> StepOutcome:
    """Chained conditionals in ``order`` (fsm.py:230-249)."""
    order = tuple(order) if order is not None else default_bundled_order(fsm)
    validate_bundled_order(fsm, order)
    return _single(fsm, k, z, 1, order)


def amortized_step(fsm: FsmDefinition, k: int, z, g=None) -> StepOutcome:
    """``step`` with the shared computation evaluated at most once (fsm.py:252-273)."""
    if g is not None:
        raise FsmError("a custom shared computation cannot run on the device")
    return _single(fsm, k, z, 2)
