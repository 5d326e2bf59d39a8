"""Batched chain drivers (drop-in for ``fsm_mcmc.lockstep``).

* :func:`init_batch` -> one ``fsmc_init`` launch: streams, starting points
  and each kernel's initial evaluation for m chains (``lockstep.py:175-206``).
* :func:`run_fsm_batched` -> ``fsmc_run``: every chain advances its own
  state machine with no barrier until it holds n samples; per-chain tick
  counters equal the reference's global ticks because the reference steps
  every chain once per tick (``lockstep.py:359-406``).  The chunked global
  stop rule and the surplus ticks the aggregate counters include are
  reproduced exactly by a second, count-only launch.
* :func:`run_standard_batched` -> ``fsmc_lockstep_run``: the lock-step
  (vmap-style) baseline built from the same device blocks.

Samples and ledgers come back as numpy arrays (``output="numpy"``, the
reference's types) or stay in HBM as torch tensors (``output="torch"``).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field
from typing import Any, Sequence

import numpy as np
import torch

from . import _lib
from .fsm import BlockFailure, ChainView, FsmDefinition, StepOutcome, default_bundled_order, \
    validate_bundled_order
from .prng import RngKey

__all__ = ["ChainBatch", "CostParams", "CostLedger", "KernelRunError", "TickBudgetExceeded",
           "init_batch", "run_standard_batched", "run_fsm_batched", "collect_samples",
           "measure_block_costs", "lockstep_barrier_us",
           "STEP_VARIANTS", "TICK_CHUNK"]

STEP_VARIANTS = ("plain", "bundled", "amortized")
TICK_CHUNK = 100
_VARIANT_ID = {"plain": _lib.PLAIN, "bundled": _lib.BUNDLED, "amortized": _lib.AMORTIZED}
_NO_LIMIT = 1 << 62


class KernelRunError(RuntimeError):
    """A kernel failed mid-run; records which chain and where (lockstep.py:50-57)."""

    def __init__(self, chain: int, iteration: int, cause: Exception):
        super().__init__(f"chain {chain}, sample index {iteration}: {cause}")
        self.chain = chain
        self.iteration = iteration
        self.cause = cause


class TickBudgetExceeded(RuntimeError):
    """The FSM loop hit its tick cap; the partial ledger is attached (lockstep.py:60-68)."""

    def __init__(self, budget: int, ledger: "CostLedger", sample_counts: list):
        super().__init__(f"tick budget {budget} exhausted with per-chain sample counts "
                         f"{sample_counts}")
        self.ledger = ledger
        self.sample_counts = sample_counts


@dataclass(frozen=True)
class CostParams:
    """Abstract block costs c_1..c_K, dispatch factor alpha and shared-site
    pricing (lockstep.py:71-155).  Host arithmetic over device counts."""

    block_costs: tuple
    alpha: float = 1.0
    loop_states: tuple = ()
    shared_cost: float = 0.0
    shared_sites: tuple = ()

    def __post_init__(self):
        if len(self.block_costs) < 1:
            raise ValueError("need at least one block cost")
        if any(c < 0 for c in self.block_costs):
            raise ValueError(f"block costs must be nonnegative: {self.block_costs}")
        if self.shared_cost < 0:
            raise ValueError("shared_cost must be nonnegative")
        sites = tuple(self.shared_sites) or (0,) * len(self.block_costs)
        if len(sites) != len(self.block_costs):
            raise ValueError("shared_sites length must match block_costs")
        object.__setattr__(self, "shared_sites", sites)
        full = self.full_block_costs()
        if sum(full) <= 0:
            raise ValueError("total block cost must be positive")
        lo = max(full) / sum(full)
        if not lo - 1e-12 <= self.alpha <= 1.0 + 1e-12:
            raise ValueError(f"alpha={self.alpha} outside admissible interval [{lo}, 1]")
        K = len(self.block_costs)
        if any(not 1 <= s <= K for s in self.loop_states):
            raise ValueError(f"loop_states {self.loop_states} outside 1..{K}")

    def full_block_costs(self) -> tuple:
        return tuple(c + s * self.shared_cost for c, s in zip(self.block_costs, self.shared_sites))

    def tick_cost(self, variant: str) -> float:
        """Charge of one executor call over the batch (lockstep.py:119-131)."""
        if variant in ("plain", "bundled"):
            return self.alpha * sum(self.full_block_costs())
        if variant == "amortized":
            extra = self.shared_cost if sum(self.shared_sites) > 0 else 0.0
            return self.alpha * sum(self.block_costs) + extra
        raise ValueError(f"unknown step variant {variant!r}")

    def shared_evals_per_tick(self, variant: str) -> int:
        if sum(self.shared_sites) == 0:
            return 0
        return int(sum(self.shared_sites)) if variant in ("plain", "bundled") else 1

    @staticmethod
    def for_fsm(fsm: FsmDefinition, block_costs=None, alpha: float = 1.0,
                shared_cost: float = 1.0) -> "CostParams":
        K = fsm.n_states
        costs = tuple(block_costs) if block_costs is not None else (1.0,) * K
        sites = tuple(fsm.shared.sites.get(k, 0) for k in range(1, K + 1)) \
            if fsm.shared is not None else (0,) * K
        return CostParams(block_costs=costs, alpha=alpha, loop_states=tuple(sorted(fsm.loop_states)),
                          shared_cost=shared_cost if fsm.shared is not None else 0.0,
                          shared_sites=sites)


@dataclass
class CostLedger:
    """Counts and model charges of one run (lockstep.py:209-228)."""

    iter_counts: Any
    loop_exec_counts: dict
    tick_count: int
    block_exec_counts: Any
    charged_cost: float
    walltime: float
    regime: str
    tick_cost: float = 0.0
    shared_evals_per_tick: int = 0
    native_shared_evals: int = 0
    sample_ticks: Any = None
    extras: dict = field(default_factory=dict)

    def cost_per_sample(self) -> float:
        return self.charged_cost / self.iter_counts.shape[0]


# ------------------------------------------------------------------ batch
class ChainBatch:
    """m chains in structure-of-arrays device state (lockstep.py:158-172).

    vec [m, n_vec, d] float64, scal [m, n_scal] float64, ints [m, 32] int64
    (counter, stream, state, tick, count, error record, block counts,
    family-private integers), err_key [1], work [256] int32 (the launch
    bookkeeping of runs on this batch: chain queues, barrier words).
    """

    def __init__(self, bundle, target, m: int, seed: int, parent_stream: int = 0,
                 chain_offset: int = 0):
        lib = _lib.lib()
        self.bundle, self.target, self.m, self.seed = bundle, target, int(m), int(seed)
        self.parent_stream, self.chain_offset = int(parent_stream), int(chain_offset)
        self.kernel = bundle.struct()
        nv, ns, nl, nk = (ctypes.c_int32() for _ in range(4))
        _lib.check(lib.fsmc_state_layout(ctypes.byref(self.kernel), target.dim, ctypes.byref(nv),
                                         ctypes.byref(ns), ctypes.byref(nl), ctypes.byref(nk)),
                   "fsmc_state_layout")
        self.n_vec, self.n_scal, self.n_loop, self.n_states = nv.value, ns.value, nl.value, nk.value
        d = target.dim
        self.vec = torch.zeros((self.m, self.n_vec, d), dtype=torch.float64, device="cuda")
        self.scal = torch.zeros((self.m, self.n_scal), dtype=torch.float64, device="cuda")
        self.ints = torch.zeros((self.m, _lib.FSMC_NINT), dtype=torch.int64, device="cuda")
        self.err_key = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        self.work = torch.zeros(_lib.WORK_WORDS, dtype=torch.int32, device="cuda")
        self.active_mask = [True] * self.m
        self._ran = False

    def struct(self, lo: int = 0, hi: int | None = None) -> _lib.State:
        hi = self.m if hi is None else hi
        s = _lib.State()
        s.m = hi - lo
        s.dim = self.target.dim
        s.n_vec, s.n_scal = self.n_vec, self.n_scal
        s.vec = self.vec[lo].data_ptr()
        s.scal = self.scal[lo].data_ptr()
        s.ints = self.ints[lo].data_ptr()
        s.seed = self.seed & ((1 << 64) - 1)
        s.err_key = self.err_key.data_ptr()
        s.work = self.work.data_ptr()
        return s

    # reference-shaped views (host copies)
    @property
    def state_ids(self) -> list:
        return self.ints[:, _lib.I_STATE].tolist()

    @property
    def sample_counts(self) -> list:
        return self.ints[:, _lib.I_COUNT].tolist()

    @property
    def locals(self) -> list:
        return [ChainView(self, j) for j in range(self.m)]

    def chain(self, j: int) -> ChainView:
        return ChainView(self, j)

    def chain_position(self, j: int) -> np.ndarray:
        return self.vec[j, 0].cpu().numpy()

    def chain_key(self, j: int) -> RngKey:
        row = self.ints[j].tolist()
        return RngKey(self.seed & ((1 << 64) - 1), row[_lib.I_STREAM] & ((1 << 64) - 1),
                      row[_lib.I_COUNTER] & ((1 << 64) - 1))

    def host_summary(self):
        """One device->host read: per chain (count, tick, error kind, error
        tick, error label, error sample index, shared evaluations) and the
        first-failure key."""
        cols = [_lib.I_COUNT, _lib.I_TICK, _lib.I_ERR_KIND, _lib.I_ERR_TICK, _lib.I_ERR_LABEL,
                _lib.I_ERR_ITER, _lib.I_SHARED]
        flat = torch.cat([self.ints[:, cols].reshape(-1), self.err_key]).cpu()
        key = int(flat[-1]) & ((1 << 64) - 1)
        return flat[:-1].reshape(self.m, len(cols)), key

    def first_error(self):
        key = int(self.err_key.item()) & ((1 << 64) - 1)
        if key == (1 << 64) - 1:
            return None
        j = key & ((1 << 24) - 1)
        row = self.ints[j].tolist()
        return (j, row[_lib.I_ERR_KIND], row[_lib.I_ERR_LABEL], row[_lib.I_ERR_TICK],
                row[_lib.I_ERR_ITER])

    def _step_one(self, j: int, k: int, variant: int, order) -> StepOutcome:
        """One executor call on chain j entering state k (fsm.step & co)."""
        K = self.n_states
        self.ints[j, _lib.I_STATE] = k
        before = self.ints[j].clone()
        tick = int(before[_lib.I_TICK])
        st = self.struct(j, j + 1)
        out = _lib.Outputs()
        ordv = (ctypes.c_int32 * K)(*(order or default_bundled_order(self.bundle.fsm)))
        self.err_key.fill_(-1)
        _lib.check(_lib.lib().fsmc_run(ctypes.byref(self.kernel), ctypes.byref(self.target.struct()),
                                       ctypes.byref(st), 0, variant, ordv, tick + 1, 1,
                                       ctypes.byref(out), 0, _lib.stream_ptr()), "fsmc_run")
        after = self.ints[j].tolist()
        if after[_lib.I_ERR_KIND] != _lib.E_NONE:
            raise _cause(self.bundle, after[_lib.I_ERR_KIND], after[_lib.I_ERR_LABEL])
        b0 = before[_lib.I_BLOCKS:_lib.I_BLOCKS + K].tolist()
        b1 = after[_lib.I_BLOCKS:_lib.I_BLOCKS + K]
        seq = list(order or default_bundled_order(self.bundle.fsm)) if variant == 1 else [k]
        executed = tuple(s for s in seq if b1[s - 1] > b0[s - 1])
        did = after[_lib.I_SHARED] > int(before[_lib.I_SHARED])
        return StepOutcome(after[_lib.I_STATE], ChainView(self, j), k == K, did, executed)


def _cause(bundle, kind: int, label: int) -> Exception:
    """Map a device error record to the reference's exception types."""
    from .kernels.base import KernelError
    labels = bundle.fsm.labels
    if kind == _lib.E_ZERO_START:
        return KernelError("starting point has zero density")
    if kind == _lib.E_GRAD:
        return KernelError("non-finite gradient")
    if kind == _lib.E_TARGET:   # targets.py:213-218
        from .targets import TargetError
        return TargetError("kernel matrix not positive definite even with jitter")
    if kind == _lib.E_INIT:     # the Locals constructor's check (e.g. drmh.py:45, slice_sampling.py:38)
        return BlockFailure(labels[0], "log-density evaluated to a non-finite value (NaN or +inf)")
    if label == _lib.SLICE_LABEL:
        name = "slice"
    else:
        name = "shared log f" if label == 0 else labels[label - 1]
    return BlockFailure(name, "log-density evaluated to a non-finite value (NaN or +inf)")


def init_batch(bundle, target, m: int, seed: int, x0=None, init_jitter: float = 0.0,
               *, parent_stream: int = 0, chain_offset: int = 0) -> ChainBatch:
    """m chains with streams split(key(seed), .) (lockstep.py:175-206).

    ``chain_offset`` selects chains [offset, offset + m) of a larger batch:
    chain j's trajectory depends only on (seed, j, target), so shards built
    this way reproduce the full batch exactly.
    """
    if m < 1:
        raise ValueError(f"need m >= 1 chains, got {m}")
    bundle.check_target(target)
    d = target.dim
    if isinstance(x0, torch.Tensor):
        x0d = x0.to(device="cuda", dtype=torch.float64).contiguous()
    else:
        x0d = torch.as_tensor(np.zeros(d) if x0 is None else np.asarray(x0, dtype=float),
                              device="cuda")
    if tuple(x0d.shape) != (d,):
        raise ValueError(f"x0 shape {tuple(x0d.shape)} does not match dim {d}")
    batch = ChainBatch(bundle, target, m, seed, parent_stream, chain_offset)
    lib = _lib.lib()
    args = (ctypes.byref(batch.kernel), ctypes.byref(target.struct()), ctypes.byref(batch.struct()),
            parent_stream & ((1 << 64) - 1), chain_offset, x0d.data_ptr(), float(init_jitter),
            _lib.stream_ptr())
    ev = None
    if hasattr(target, "batched_evaluator") and bundle.family != _lib.NUTS:
        ev = target.batched_evaluator(bundle.family)
    if ev is None:
        _lib.check(lib.fsmc_init(*args), "fsmc_init")
    else:
        # starting points evaluated in one batched call (fsmc_init_deferred/_finish)
        _lib.check(lib.fsmc_init_deferred(*args), "fsmc_init_deferred")
        X = batch.vec[:, 0, :].contiguous()
        lp = torch.empty(m, dtype=torch.float64, device="cuda")
        ev(X, lp, None)
        _lib.check(lib.fsmc_init_finish(ctypes.byref(batch.kernel), ctypes.byref(target.struct()),
                                        ctypes.byref(batch.struct()), lp.data_ptr(),
                                        _lib.stream_ptr()), "fsmc_init_finish")
    err = batch.first_error()
    if err is not None:
        raise _cause(bundle, err[1], err[2])
    return batch


def _validate_run_args(batch: ChainBatch, n: int):
    if n < 1:
        raise ValueError(f"need n >= 1 samples, got {n}")
    if batch._ran:   # lockstep.py:231-235 (a batch is fresh until a driver runs it)
        raise ValueError("batch has already been run; build a fresh one")


def _outputs(n, m, d, L, want_ticks, want_samples=True, counts64=False):
    """Device outputs; counts64: the loop counts in int64 (the reference's
    ledger type) so they can go to the host without a conversion."""
    # every row < n of every chain is written by the kernel before it is read
    samples = torch.empty((n, m, d), dtype=torch.float64, device="cuda") if want_samples else None
    loops = torch.empty((L, n, m), dtype=torch.int64 if counts64 else torch.int32, device="cuda")
    ticks = torch.empty((n, m), dtype=torch.int32, device="cuda") if want_ticks else None
    out = _lib.Outputs()
    out.samples = _lib.ptr(samples)
    if counts64:
        out.loop_counts64 = loops.data_ptr()
    else:
        out.loop_counts = loops.data_ptr()
    out.sample_ticks = _lib.ptr(ticks)
    return samples, loops, ticks, out


def _pinned(shape, dtype):
    """Page-locked host buffer (torch's caching host allocator: reused across
    runs once freed), so device-to-host copies run at full link speed and can
    be asynchronous."""
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def _to_host(x, dtype=None):
    """Asynchronous copy of a device tensor into pinned host memory (converted
    on the device first when `dtype` differs); the caller synchronises."""
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    h = _pinned(tuple(x.shape), x.dtype)
    h.copy_(x, non_blocking=True)
    return h


def _convert(x, output):
    if x is None:
        return None
    if output == "torch":
        return x
    h = _to_host(x)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def _counts(x, output):
    """Ledger count matrices: int64 numpy arrays (the reference's type) for
    output="numpy" (widened on the device, one pinned copy); int32 device
    tensors, unconverted, for output="torch"."""
    if output == "torch":
        return x
    h = _to_host(x, torch.int64)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def run_fsm_batched(bundle, target, batch: ChainBatch, n: int, step_variant: str = "plain",
                    cost_params: CostParams | None = None, tick_budget: int | None = None,
                    bundled_order: tuple | None = None, record_sample_ticks: bool = False,
                    tick_chunk: int = TICK_CHUNK, *, surplus: bool = True, output: str = "numpy",
                    lanes: int = 0, evaluator=None, draw_window: int = 0,
                    prior_transform=None, draw_parts: int = 1, prior_parts: int = 1,
                    stop_sync=None, precision: str = "fp64", _timing: dict | None = None):
    """Run every chain's machine until each holds n samples (lockstep.py:308-416).

    ``surplus=False`` skips the reference's surplus ticks (steps of chains
    that already hold n samples, discarded by the reference): samples and
    every per-sample ledger field are unchanged, only the two aggregate
    counters then stop at each chain's n-th sample.

    ``evaluator``: batched-evaluation mode.  Chains advance to their next
    log-density request (``fsmc_advance``); all requests of a round are then
    evaluated in one call ``evaluator(theta[k, d], lp[k], grad[k, d] | None)``
    -- e.g. GEMMs across chains for a dense target -- and the chains resume.
    ``evaluator="device"`` uses the per-point device plugin (bit-identical
    to the default mode).  Targets whose ``batched_evaluator()`` is not None
    (large dense designs) use it automatically.

    ``prior_transform`` (elliptical kernel with a dense Gaussian prior):
    batch the INIT block's nu = L eps across chains (``fsmc_advance_prior``).
    Chains run with the plugin evaluated in place until their next INIT,
    park eps, and all parked rows are transformed in one call.  "dmma": the
    hand-written fp64 tensor-core triangular product (``fsmc_prior_trmm``;
    values within its rounding); "gemm": one fp64 GEMM ``eps @ L^T`` (cuBLAS
    DGEMM); "trmm": the same product as a triangular cuBLAS DTRMM;
    "device": ``fsmc_prior_apply``, the sampling kernel's summation order
    (bit-identical to the default mode); or a callable ``f(nu[k, d])``
    transforming the rows in place.  ``prior_parts`` (1..8) splits the chains
    in parts whose rounds overlap on their own streams.

    ``precision="fp32"``: the throughput mode -- chain state and arithmetic
    in fp32 (the draws are still the reference's fp64 values, each rounded
    once; the HBM state and the samples stay float64).  Distributional
    parity only (tests/test_gpu_distribution.py); compiled for DRMH on the
    MoG / funnel (d <= 10) and NUTS on the equicorrelated Gaussian.

    ``stop_sync`` (a sharded batch, ``distributed.stop_sync(group)``): the
    stop tick, completion and first failure are reduced over every rank's
    shard, so ``tick_count``, the surplus ticks behind the aggregate
    counters and the raised failure are the whole batch's (chain indices
    global); ``distributed.global_ledger`` then merges the shard ledgers.

    ``draw_window`` (DRMH kernels): generate each chain's next ``draw_window``
    PRNG draws in a separate full-occupancy kernel and let the step kernel
    read them (``fsmc_run_windowed``); bit-identical to the inline draws.
    ``draw_parts`` (1..16) splits the chains in parts whose generator and
    step kernels overlap on their own streams (``fsmc_run_windowed_overlap``);
    ``draw_parts=0`` pipelines the windows instead: every window runs each
    chain exactly ``draw_window // (dim + 1)`` proposals, so window r + 1 is
    generated (double-buffered) while window r runs, all chains in one launch.
    """
    _validate_run_args(batch, n)
    bundle.check_target(target)
    if step_variant not in STEP_VARIANTS:
        raise ValueError(f"step_variant must be one of {STEP_VARIANTS}")
    if output not in ("numpy", "torch"):
        raise ValueError("output must be 'numpy' or 'torch'")
    params = cost_params or bundle.default_costs
    machine = bundle.fsm
    K = machine.n_states
    if len(params.block_costs) != K:
        raise ValueError(f"{len(params.block_costs)} block costs for a {K}-state kernel")
    order = tuple(bundled_order or default_bundled_order(machine))
    if step_variant == "bundled":
        validate_bundled_order(machine, order)
    m, d = batch.m, target.dim
    loop_states = bundle.loop_states
    to_host = output == "numpy"
    samples, loops, ticks_out, out = _outputs(n, m, d, len(loop_states), record_sample_ticks,
                                              counts64=to_host)
    # output="numpy": the samples and the ledger's count matrices land in
    # pinned host memory; the per-chain and windowed runs stream finished rows
    # / chain parts out while they sample (fsmc_run_egress, fsmc_run_windowed_egress)
    host = _pinned((n, m, d), torch.float64) if to_host else None
    eg = None
    host_counts = host_iter = None
    if to_host:
        host_counts = _pinned((len(loop_states), n, m), torch.int64)
        eg = _lib.Egress()
        eg.samples = host.data_ptr()
        eg.loop_counts = host_counts.data_ptr()
        eg.n_loops = len(loop_states)
        if len(bundle.iter_states) == 1:
            host_iter = _pinned((n, m), torch.int64)
            eg.iter_counts = host_iter.data_ptr()
            eg.iter_loop = loop_states.index(bundle.iter_states[0])
    egressed = False
    counts_egressed = False
    limit = (tick_budget // tick_chunk) * tick_chunk if tick_budget is not None else _NO_LIMIT
    lib = _lib.lib()
    if precision not in ("fp64", "fp32"):
        raise ValueError("precision must be 'fp64' or 'fp32'")
    kern, tgt = batch.kernel, target.struct()
    if precision == "fp32":
        if evaluator is not None or prior_transform is not None:
            raise ValueError("the fp32 throughput mode runs the per-chain plugins only")
        kern = _lib.Kernel.from_buffer_copy(batch.kernel)
        kern.precision = 1
    ordv = (ctypes.c_int32 * K)(*order)
    variant = _VARIANT_ID[step_variant]

    if evaluator is None and hasattr(target, "batched_evaluator"):
        evaluator = target.batched_evaluator(bundle.family)
    if draw_window and (bundle.family != _lib.DRMH or evaluator is not None):
        raise ValueError("draw_window applies to the DRMH kernels without an evaluator")
    if prior_transform is not None:
        gp = getattr(target, "gaussian_prior", None)
        if bundle.family != _lib.ESS or gp is None or evaluator is not None or draw_window:
            raise ValueError("prior_transform applies to the elliptical kernel with a Gaussian "
                             "prior, without an evaluator")
        if target.struct().prior_kind != _lib.PRIOR_DENSE:
            prior_transform = None      # identity prior: nu = eps, nothing to batch
    if prior_transform is not None:
        launch = _prior_launcher(target, batch, n, variant, ordv, out, lanes, prior_transform,
                                 prior_parts, samples, host)
        egressed = host is not None
    elif draw_window:
        # [m][window] plus a line of slack: the step kernel prefetches the
        # next proposal's draws, which for the last chain may lie past its window
        # (draw_parts=0: two windows per chain, the double buffer)
        nbuf = 2 if int(draw_parts) == 0 else 1
        draws = torch.empty(nbuf * m * int(draw_window) + 32, dtype=torch.float64, device="cuda")

        def launch(mode, tick_limit):
            nonlocal egressed, counts_egressed
            dst = ctypes.byref(eg) if eg is not None and mode == 0 else None
            _lib.check(lib.fsmc_run_windowed_egress(ctypes.byref(kern), ctypes.byref(tgt),
                                                    ctypes.byref(batch.struct()), n, variant, ordv,
                                                    tick_limit, mode, ctypes.byref(out),
                                                    int(draw_window), draws.data_ptr(), lanes,
                                                    int(draw_parts), dst, _lib.stream_ptr()),
                       "fsmc_run_windowed_egress")
            egressed = egressed or dst is not None
            counts_egressed = counts_egressed or dst is not None
    elif evaluator is None:
        def launch(mode, tick_limit):
            nonlocal egressed, counts_egressed
            dst = ctypes.byref(eg) if eg is not None and mode == 0 else None
            # chains in parts: each finished part's samples and counts stream
            # to the host while the next parts run
            parts = max(1, min(_EGRESS_PARTS_MAX, m // _EGRESS_PART_CHAINS)) if dst else 1
            _lib.check(lib.fsmc_run_egress(ctypes.byref(kern), ctypes.byref(tgt),
                                           ctypes.byref(batch.struct()), n, variant, ordv, tick_limit,
                                           mode, ctypes.byref(out), lanes, parts, dst,
                                           _lib.stream_ptr()), "fsmc_run_egress")
            egressed = egressed or dst is not None
            counts_egressed = counts_egressed or dst is not None
    else:
        launch = _batched_launcher(bundle, target, batch, n, variant, ordv, out, lanes, evaluator)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if _timing is not None:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
    launch(0, limit)
    if _timing is not None:
        ev[1].record()
    info, key = batch.host_summary()          # one device->host read
    counts, cticks = info[:, 0], info[:, 1]
    errored = info[:, 2] != _lib.E_NONE
    all_done = bool((counts >= n).all())
    if all_done:
        tick_count = -(-int(cticks.max()) // tick_chunk) * tick_chunk
    else:
        tick_count = limit
    first_err = int(info[errored, 3].min()) if bool(errored.any()) else _NO_LIMIT
    g_err = None
    if stop_sync is not None:
        # sharded batch: the reference's stop rule is global (lockstep.py:359-366)
        tick_count, all_done, g_key, g_rec = stop_sync(*_shard_stop(batch, info, key, tick_count,
                                                                    all_done))
        if not all_done:
            tick_count = limit
        first_err = g_key >> 24 if g_key < _NO_LIMIT else _NO_LIMIT
    run_to = min(tick_count, first_err)
    if run_to < _NO_LIMIT and (surplus or first_err < _NO_LIMIT) and int(cticks.min()) < run_to:
        launch(1, run_to)
        info, key = batch.host_summary()
    else:
        torch.cuda.synchronize()
    if stop_sync is not None:
        # the surplus ticks may have failed earlier than any failure seen so far
        _, _, g_key, g_rec = stop_sync(*_shard_stop(batch, info, key, tick_count, all_done))
        if g_key < _NO_LIMIT:
            g_err = (g_key, g_rec)
    walltime = time.perf_counter() - t0
    if _timing is not None:
        _timing["run_kernel_ms"] = ev[0].elapsed_time(ev[1])
    batch.active_mask = [False] * m
    batch._ran = True

    if g_err is not None:
        (g_key, (kind, label, eiter)) = g_err
        if (g_key >> 24) <= tick_count:
            raise KernelRunError(chain=g_key & ((1 << 24) - 1), iteration=eiter,
                                 cause=_cause(bundle, kind, label))
    elif stop_sync is None and key != (1 << 64) - 1:
        j = key & ((1 << 24) - 1)
        kind, etick_j, label, eiter = (int(v) for v in info[j, 2:6])
        if etick_j <= tick_count:
            raise KernelRunError(chain=j, iteration=eiter, cause=_cause(bundle, kind, label))
    counts_now = info[:, 0]
    n_done = n if all_done else int(counts_now.min())
    streamed = (host_counts, host_iter) if counts_egressed and n_done == n else None
    ledger = _fsm_ledger(bundle, params, step_variant, batch, loops, ticks_out, n_done,
                         tick_count if all_done else limit, walltime, output,
                         native_shared=int(info[:, 6].sum()), streamed=streamed)
    if hasattr(launch, "stats"):
        ledger.extras.update(launch.stats)
    if not all_done:
        raise TickBudgetExceeded(tick_budget, ledger, counts_now.tolist())
    if host is None:
        return samples, ledger
    if not egressed:
        host.copy_(samples, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy(), ledger


def _shard_stop(batch, info, key, tick_count, all_done):
    """This shard's stop-rule fields for distributed.stop_sync: the chunked
    stop tick, completion, and its first failure as a key over global chain
    indices (tick << 24 | chain_offset + j) with (kind, label, sample index)."""
    if key == (1 << 64) - 1:
        return tick_count, all_done, _NO_LIMIT, (0, 0, 0)
    j = key & ((1 << 24) - 1)
    kind, etick, label, eiter = (int(v) for v in info[j, 2:6])
    return tick_count, all_done, (etick << 24) | (batch.chain_offset + j), (kind, label, eiter)


def _device_evaluator(target, family: int, lanes: int):
    """Per-point device plugin over the request list (fsmc_target_eval), in
    the sampling kernel's lane layout (same reduction order)."""
    tgt = target.struct()

    def evaluate(theta, lp, g):
        k = theta.shape[0]
        _lib.check(_lib.lib().fsmc_target_eval(ctypes.byref(tgt), theta.data_ptr(), k, lp.data_ptr(),
                                               _lib.ptr(g), family, lanes, _lib.stream_ptr()),
                   "fsmc_target_eval")
    return evaluate


def _batched_launcher(bundle, target, batch, n, variant, ordv, out, lanes, evaluator):
    """Rounds of fsmc_advance + one batched evaluation of every request."""
    m, d = batch.m, target.dim
    grad = bundle.family == _lib.NUTS
    if evaluator == "device":
        evaluator = _device_evaluator(target, bundle.family, lanes)
    theta = torch.empty((m, d), dtype=torch.float64, device="cuda")
    lp = torch.empty(m, dtype=torch.float64, device="cuda")
    g = torch.empty((m, d), dtype=torch.float64, device="cuda") if grad else None
    req_chain = torch.empty(m, dtype=torch.int32, device="cuda")
    req_count = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib = _lib.lib()
    kern, tgt = batch.kernel, target.struct()
    stats = {"rounds": 0, "evaluations": 0}

    def launch(mode, tick_limit):
        while True:
            _lib.check(lib.fsmc_advance(ctypes.byref(kern), ctypes.byref(tgt),
                                        ctypes.byref(batch.struct()), n, variant, ordv, tick_limit,
                                        mode, ctypes.byref(out), lp.data_ptr(), _lib.ptr(g),
                                        theta.data_ptr(), req_chain.data_ptr(),
                                        req_count.data_ptr(), lanes, _lib.stream_ptr()),
                       "fsmc_advance")
            k = int(req_count.item())
            if k == 0:
                return
            stats["rounds"] += 1
            stats["evaluations"] += k
            evaluator(theta[:k], lp[:k], None if g is None else g[:k])

    launch.stats = stats
    return launch


_SIDE_STREAMS: dict = {}      # per device, reused across runs (prior_parts)
# per-chain runs with host output (fsmc_run_egress): chain parts of at least
# this many chains, at most this many parts; each finished part's columns go
# to the host while later parts run, so the copy left after the run is one
# part's (C3 e2e: 5.40e7 at 8 parts of 2048 chains, 5.71e7 at 16 of 1024)
_EGRESS_PART_CHAINS = int(os.environ.get("FSMC_EGRESS_PART_CHAINS", "1024"))
_EGRESS_PARTS_MAX = int(os.environ.get("FSMC_EGRESS_PARTS_MAX", "16"))
_EGRESS_STREAMS: dict = {}    # per device: device -> host sample copies


def _prior_launcher(target, batch, n, variant, ordv, out, lanes, transform, parts=1,
                    samples=None, host=None):
    """Rounds of fsmc_advance_prior + one batched nu = L eps over every
    chain parked at INIT.  parts > 1: the chains in contiguous parts, each
    with its own rounds on its own stream (fsmc_advance_prior_part), so one
    part's transform overlaps another part's advance kernel.

    ``host`` (pinned, output="numpy"): a round completes one sample of every
    chain of its part (each chain runs from one INIT park to the next), so
    after a part's t-th advance its sample rows [0, t) are final and go to
    the host (one pitched copy per round) on an egress stream while the
    rounds continue."""
    m, d = batch.m, target.dim
    parts = max(1, min(int(parts), 8, m))
    bounds = [(m * h // parts, m * (h + 1) // parts) for h in range(parts)]
    nu = torch.empty((m, d), dtype=torch.float64, device="cuda")
    req_chain = torch.empty(m, dtype=torch.int32, device="cuda")
    req_count = torch.zeros(parts, dtype=torch.int32, device="cuda")
    lib = _lib.lib()
    kern, tgt = batch.kernel, target.struct()
    if transform in ("gemm", "trmm", "dmma"):
        from .dense import PriorTransform
        transform = [PriorTransform(target.device_arrays()["prior_t"], transform, target)
                     for _ in range(parts)]
        for h, t in enumerate(transform):    # scratch allocated up front, on this stream
            t.tmp = torch.empty((bounds[h][1] - bounds[h][0], d), dtype=torch.float64, device="cuda")
    elif transform == "device":
        def transform(rows):
            _lib.check(lib.fsmc_prior_apply(ctypes.byref(tgt), rows.data_ptr(), rows.shape[0],
                                            _lib.stream_ptr()), "fsmc_prior_apply")
    elif not callable(transform):
        raise ValueError("prior_transform must be 'dmma', 'trmm', 'gemm', 'device' or a callable")
    if not isinstance(transform, list):
        transform = [transform] * parts
    stats = {"rounds": 0, "prior_transforms": 0}
    main = torch.cuda.current_stream()
    side = _SIDE_STREAMS.setdefault(main.device, [])
    while len(side) < parts - 1:
        side.append(torch.cuda.Stream(device=main.device))
    streams = [main] + side[:parts - 1]

    def advance(h, mode, tick_limit):
        lo, hi = bounds[h]
        _lib.check(lib.fsmc_advance_prior_part(
            ctypes.byref(kern), ctypes.byref(tgt), ctypes.byref(batch.struct()), n, variant, ordv,
            tick_limit, mode, ctypes.byref(out), nu[lo:].data_ptr(), req_chain[lo:].data_ptr(),
            req_count[h:].data_ptr(), lanes, lo, hi, h, _lib.stream_ptr()),
            "fsmc_advance_prior_part")

    egress = _EGRESS_STREAMS.setdefault(main.device, torch.cuda.Stream(device=main.device)) \
        if host is not None else None
    pitch = m * d * 8

    def send(h, upto, sent):
        """rows [sent[h], upto) of part h's chain columns to the host"""
        if egress is None or upto <= sent[h]:
            return
        lo, hi = bounds[h]
        off = sent[h] * pitch + lo * d * 8
        _lib.check(lib.fsmc_copy_to_host_2d(host.data_ptr() + off, samples.data_ptr() + off, pitch,
                                            (hi - lo) * d * 8, upto - sent[h], egress.cuda_stream),
                   "fsmc_copy_to_host_2d")
        sent[h] = upto

    # one pinned completion word per part and round parity: a part's rounds are
    # issued without waiting for the host, and its parked-chain count is read
    # one round late (at most one extra, empty round per part at the end)
    counts_h = torch.zeros((parts, 2), dtype=torch.int32, pin_memory=True)
    done_ev = [[torch.cuda.Event() for _ in range(2)] for _ in range(parts)]

    def issue(h, mode, tick_limit, r):
        """round r of part h on its stream: (transform, when r > 0) + advance,
        then its parked-chain count to pinned memory"""
        lo, hi = bounds[h]
        if r > 0:
            transform[h](nu[lo:hi])
        advance(h, mode, tick_limit)
        counts_h[h, r & 1].copy_(req_count[h], non_blocking=True)
        done_ev[h][r & 1].record()

    def launch(mode, tick_limit):
        for s in streams[1:]:
            s.wait_stream(main)
        if egress is not None:
            egress.wait_stream(main)
        sent = [0] * parts
        rounds = [0] * parts         # rounds issued per part
        active = list(range(parts))
        for h in active:
            with torch.cuda.stream(streams[h]):
                issue(h, mode, tick_limit, 0)
                rounds[h] = 1
        while active:
            still = []
            for h in active:
                with torch.cuda.stream(streams[h]):
                    r = rounds[h]
                    # round r (transform of round r-1's parks + advance) goes
                    # out before round r-1's count is read
                    issue(h, mode, tick_limit, r)
                    rounds[h] = r + 1
                    done_ev[h][(r - 1) & 1].synchronize()
                    k = int(counts_h[h, (r - 1) & 1])
                    if mode == 0 and egress is not None:
                        # after round r-1 (the part's r-th advance) rows [0, r-1) are final
                        egress.wait_event(done_ev[h][(r - 1) & 1])
                        send(h, min(r - 1, n), sent)
                    if k == 0:
                        if mode == 0 and egress is not None:
                            egress.wait_stream(streams[h])
                            send(h, n, sent)
                        continue
                    stats["rounds"] += 1
                    stats["prior_transforms"] += k
                    still.append(h)
            active = still
        for s in streams[1:]:
            main.wait_stream(s)
        if egress is not None:
            main.wait_stream(egress)

    launch.stats = stats
    return launch


def _fsm_ledger(bundle, params, variant, batch, loops, ticks_out, n_rows, ticks, walltime,
                output, native_shared: int, streamed=None) -> CostLedger:
    """lockstep.py:419-451.  ``streamed``: the count matrices already in
    pinned host memory (int64 loop counts [L][n][m], iter_counts [n][m] or
    None), copied there during the run."""
    K = bundle.fsm.n_states
    loop_states = bundle.loop_states
    if streamed is not None:
        torch.cuda.current_stream().synchronize()
        hc, hi = streamed
        loop_execs = {s: hc[i].numpy() for i, s in enumerate(loop_states)}
    else:
        loop_execs = {s: _counts(loops[i, :n_rows], output) for i, s in enumerate(loop_states)}
    its = [loops[loop_states.index(s), :n_rows] for s in bundle.iter_states]
    it = its[0] if len(its) == 1 else sum(t.to(torch.int64) for t in its)
    blocks = batch.ints[:, _lib.I_BLOCKS:_lib.I_BLOCKS + K].sum(0)
    tc = params.tick_cost(variant)
    st = None if ticks_out is None else _counts(ticks_out[:n_rows], output)
    return CostLedger(
        iter_counts=streamed[1].numpy() if streamed is not None and streamed[1] is not None
        else _counts(it, output),
        loop_exec_counts=loop_execs, tick_count=int(ticks),
        block_exec_counts=_convert(blocks, output), charged_cost=ticks * tc, walltime=walltime,
        regime=f"fsm-{variant}", tick_cost=tc,
        shared_evals_per_tick=params.shared_evals_per_tick(variant),
        native_shared_evals=native_shared, sample_ticks=st)


def run_standard_batched(bundle, target, batch: ChainBatch, n: int,
                         cost_params: CostParams | None = None, *, output: str = "numpy",
                         lanes: int = 0, evaluator=None):
    """Lock-step baseline: one monolithic sample per chain per iteration with
    barrier semantics (lockstep.py:238-305), on the device.

    ``evaluator``: the lock-step baseline of the batched-evaluation mode
    (``fsmc_advance_lockstep``): every round evaluates one point per chain in
    one call, and no chain starts its next sample until all chains finished
    the current one (chains waiting at the barrier submit idle points, as a
    vmapped while loop evaluates the whole batch).  Same evaluator contract
    as ``run_fsm_batched``; "device" = the per-point plugin."""
    _validate_run_args(batch, n)
    bundle.check_target(target)
    params = cost_params or bundle.default_costs
    fsm = bundle.fsm
    K = fsm.n_states
    loop_states = tuple(sorted(params.loop_states or fsm.loop_states))
    if not set(loop_states) <= fsm.loop_states:
        raise ValueError(f"cost loop_states {loop_states} are not loop states of the kernel")
    full = params.full_block_costs()
    if len(full) != K:
        raise ValueError(f"{len(full)} block costs for a {K}-state kernel")
    nonloop_cost = sum(c for s, c in zip(range(1, K + 1), full) if s not in loop_states)
    m, d = batch.m, target.dim
    rec = bundle.loop_states
    samples, loops, _, out = _outputs(n, m, d, len(rec), False)
    if evaluator is None and hasattr(target, "batched_evaluator"):
        evaluator = target.batched_evaluator(bundle.family)
    stats = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if evaluator is None:
        _lib.check(_lib.lib().fsmc_lockstep_run(ctypes.byref(batch.kernel),
                                                ctypes.byref(target.struct()),
                                                ctypes.byref(batch.struct()), n, ctypes.byref(out),
                                                lanes, _lib.stream_ptr()), "fsmc_lockstep_run")
    else:
        stats = _lockstep_batched(bundle, target, batch, n, out, lanes, evaluator)
    torch.cuda.synchronize()
    walltime = time.perf_counter() - t0
    batch.active_mask = [False] * m
    batch._ran = True
    errs = batch.ints[:, [_lib.I_ERR_KIND, _lib.I_ERR_ITER]].cpu()
    bad = (errs[:, 0] != _lib.E_NONE).nonzero().flatten().tolist()
    if bad:
        j = min(bad, key=lambda c: (int(errs[c, 1]), c))
        row = batch.ints[j].tolist()
        raise KernelRunError(chain=j, iteration=row[_lib.I_ERR_ITER],
                             cause=_cause(bundle, row[_lib.I_ERR_KIND], row[_lib.I_ERR_LABEL]))
    L64 = loops.to(torch.int64)
    charged = float(n) * nonloop_cost
    if loop_states:
        mx = L64.max(dim=2).values.to(torch.float64).cpu().numpy()   # [L, n]
        for s in loop_states:
            charged += full[s - 1] * float(mx[rec.index(s)].sum())
    loop_execs = {s: _convert(L64[i], output) for i, s in enumerate(rec)}
    it = sum(L64[rec.index(s)] for s in bundle.iter_states)
    blocks = batch.ints[:, _lib.I_BLOCKS:_lib.I_BLOCKS + K].sum(0)
    ledger = CostLedger(iter_counts=_convert(it, output), loop_exec_counts=loop_execs,
                        tick_count=n, block_exec_counts=_convert(blocks, output),
                        charged_cost=charged, walltime=walltime, regime="standard")
    if stats is not None:
        ledger.extras.update(stats)
    return _convert(samples, output), ledger


def lockstep_barrier_us(bundle, target, batch: ChainBatch, iters: int = 4000,
                        lanes: int = 0) -> float:
    """Microseconds per grid-wide barrier of the lock-step baseline for this
    batch's configuration (``fsmc_lockstep_barrier_probe``: the same
    cooperative grid as ``run_standard_batched``, barriers only).  Every
    while-loop test of the lock-step run is one such barrier, so
    (tests x this) is the synchronisation share of its time."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    args = (ctypes.byref(batch.kernel), ctypes.byref(target.struct()), ctypes.byref(batch.struct()))
    _lib.check(_lib.lib().fsmc_lockstep_barrier_probe(*args, 16, lanes, _lib.stream_ptr()),
               "fsmc_lockstep_barrier_probe")          # warm-up
    ev[0].record()
    _lib.check(_lib.lib().fsmc_lockstep_barrier_probe(*args, int(iters), lanes, _lib.stream_ptr()),
               "fsmc_lockstep_barrier_probe")
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3 / iters


def _lockstep_batched(bundle, target, batch, n, out, lanes, evaluator) -> dict:
    """Rounds of fsmc_advance_lockstep + one batched evaluation each."""
    m, d = batch.m, target.dim
    if evaluator == "device":
        evaluator = _device_evaluator(target, bundle.family, lanes)
    grad = bundle.family == _lib.NUTS
    theta = torch.empty((m, d), dtype=torch.float64, device="cuda")
    lp = torch.empty(m, dtype=torch.float64, device="cuda")
    g = torch.empty((m, d), dtype=torch.float64, device="cuda") if grad else None
    req_chain = torch.empty(m, dtype=torch.int32, device="cuda")
    req_count = torch.zeros(1, dtype=torch.int32, device="cuda")
    level = torch.zeros(3, dtype=torch.int64, device="cuda")
    lib = _lib.lib()
    kern, tgt = batch.kernel, target.struct()
    stats = {"rounds": 0, "evaluations": 0}
    while True:
        _lib.check(lib.fsmc_advance_lockstep(ctypes.byref(kern), ctypes.byref(tgt),
                                             ctypes.byref(batch.struct()), n, ctypes.byref(out),
                                             lp.data_ptr(), _lib.ptr(g), theta.data_ptr(),
                                             req_chain.data_ptr(), req_count.data_ptr(),
                                             level.data_ptr(), lanes, _lib.stream_ptr()),
                   "fsmc_advance_lockstep")
        k = int(req_count.item())
        if k == 0:
            return stats
        if int(level[2].item()) == 0:   # only idle requests: the barrier opens, no evaluation
            continue
        stats["rounds"] += 1
        stats["evaluations"] += k
        evaluator(theta[:k], lp[:k], None if g is None else g[:k])


def measure_block_costs(bundle, target, m: int = 8, seed: int = 0, ticks: int = 200) -> CostParams:
    """Per-block costs from the device's own clock (lockstep.py:454-498).

    One ``fsmc_profile_blocks`` launch runs ``ticks`` plain ticks of m fresh
    chains with clock64() around every block and every log-density
    evaluation.  The launch's wall time (CUDA events) is apportioned to the
    states by their cycle shares, so a cost is the seconds of batch time one
    execution accounts for at this occupancy.  With a shared computation the
    evaluations are priced separately (``shared_cost``), as the reference
    times ``shared.fn``; otherwise they stay inside their block.  Measured
    costs vary run to run, as the reference's do."""
    batch = init_batch(bundle, target, m, seed)
    machine = bundle.fsm
    K = machine.n_states
    cycles = torch.zeros(16, dtype=torch.int64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    _lib.check(_lib.lib().fsmc_profile_blocks(ctypes.byref(batch.kernel),
                                              ctypes.byref(target.struct()),
                                              ctypes.byref(batch.struct()), int(ticks),
                                              cycles.data_ptr(), _lib.stream_ptr()),
               "fsmc_profile_blocks")
    ev[1].record()
    torch.cuda.synchronize()
    batch._ran = True
    err = batch.first_error()
    if err is not None:
        raise KernelRunError(chain=err[0], iteration=err[4], cause=_cause(bundle, err[1], err[2]))
    seconds = ev[0].elapsed_time(ev[1]) / 1e3
    cyc = [int(v) & ((1 << 64) - 1) for v in cycles.cpu().tolist()]
    blk, evc = cyc[:K], cyc[8:8 + K]
    counts = batch.ints[:, _lib.I_BLOCKS:_lib.I_BLOCKS + K].sum(0).tolist()
    shared_evals = int(batch.ints[:, _lib.I_SHARED].sum())
    per_cycle = seconds / max(1, sum(blk) + sum(evc))
    if machine.shared is not None:
        block_costs = tuple(blk[k] * per_cycle / counts[k] if counts[k] else 0.0 for k in range(K))
        shared_cost = sum(evc) * per_cycle / shared_evals if shared_evals else 0.0
        sites = tuple(machine.shared.sites.get(s, 0) for s in range(1, K + 1))
    else:
        block_costs = tuple((blk[k] + evc[k]) * per_cycle / counts[k] if counts[k] else 0.0
                            for k in range(K))
        shared_cost, sites = 0.0, (0,) * K
    return CostParams(block_costs=block_costs, alpha=1.0, loop_states=tuple(sorted(machine.loop_states)),
                      shared_cost=shared_cost, shared_sites=sites)


def collect_samples(buffers: Sequence[Sequence], flags=None, n: int | None = None) -> list:
    """Filter per-chain trace buffers to their flagged entries (lockstep.py:501-526)."""
    out = []
    for j, buf in enumerate(buffers):
        if flags is None:
            vals = list(buf)
        else:
            fl = flags[j]
            if len(fl) != len(buf):
                raise ValueError(f"chain {j}: {len(fl)} flags for {len(buf)} buffered values")
            vals = [v for v, f in zip(buf, fl) if f]
        if n is not None:
            if len(vals) < n:
                raise ValueError(f"chain {j}: only {len(vals)} samples, need {n}")
            vals = vals[:n]
        out.append(np.asarray(vals))
    return out
