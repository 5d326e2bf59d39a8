"""Chain sharding across GPUs (one process per GPU, torch.distributed).

Chains are independent (``prng.py:84-94``): rank r of W owns the contiguous
chains [r*m/W, (r+1)*m/W) and runs them with no data-path collective.  The
only cross-rank traffic is small and happens at the end of a run (NCCL over
NVLink on GPUs, gloo in the CPU tests):

* the global stop rule (``lockstep.py:359-366``): every rank's chunked stop
  tick, completion flag and first-failure key are reduced once after the
  sampling launch (:func:`stop_sync`), so the surplus ticks the reference's
  aggregate counters include run to the same global tick on every shard and
  the first failure in (tick, chain) order is raised on every rank;
* :func:`global_ledger`: the per-sample count matrices gathered along the
  chain axis (N_ij for ``efficiency_report`` / ``bound_R``), aggregate counters
  summed, ``tick_count`` / walltime as the max;
* the diagnostics' partial moments (:func:`allreduce_moments`): chain-mean
  sums, the spread of chain means (two-pass, no cancellation), max chain
  variance, and lag tiles of summed autocovariances fetched only as far as
  Geyer's truncation needs, or every lag at once.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .analysis import LAG_TILE, DiagMoments

__all__ = ["shard_range", "allreduce_moments", "LocalMoments", "stop_sync", "global_ledger"]


def shard_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous chain range of one rank."""
    return (m * rank) // world, (m * (rank + 1)) // world


class LocalMoments:
    """One rank's raw partials: n rows, chain means [m_local, d], tile(k) -> [32, d],
    and optionally all(): every lag [n, d]."""

    def __init__(self, n: int, chain_means: np.ndarray, max_chain_var: np.ndarray, acov_tile,
                 acov_all=None):
        self.n = n
        self.chain_means = np.asarray(chain_means, dtype=np.float64)
        self.max_chain_var = np.asarray(max_chain_var, dtype=np.float64)
        self.acov_tile = acov_tile
        self.acov_all = acov_all


def _allreduce(arr: np.ndarray, op, device) -> np.ndarray:
    t = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64), device=device)
    dist.all_reduce(t, op=op)
    return t.cpu().numpy()


def allreduce_moments(local: LocalMoments, device="cpu") -> DiagMoments:
    """Combine every rank's partials into global DiagMoments.

    Collectives: sum of (m_local, sum of means), then sum of squared
    deviations of chain means about the global mean, max of chain variances,
    and one sum per lag tile on demand.  Every rank must call acov_tile(k)
    for the same k sequence (the Geyer loop is deterministic given the
    all-reduced values, so it is).
    """
    m_loc, d = local.chain_means.shape
    head = np.concatenate([[float(m_loc)], local.chain_means.sum(axis=0)])
    head = _allreduce(head, dist.ReduceOp.SUM, device)
    M = int(round(head[0]))
    gmean = head[1:] / M
    ss = _allreduce(((local.chain_means - gmean) ** 2).sum(axis=0), dist.ReduceOp.SUM, device)
    var_means = ss / (M - 1) if M > 1 else np.zeros(d)
    mx = _allreduce(local.max_chain_var, dist.ReduceOp.MAX, device)

    def tile(k: int) -> np.ndarray:
        return _allreduce(local.acov_tile(k), dist.ReduceOp.SUM, device)

    def every_lag() -> np.ndarray:
        return _allreduce(local.acov_all(), dist.ReduceOp.SUM, device)

    return DiagMoments(n=local.n, m=M, d=d, var_means=var_means, max_chain_var=mx,
                       acov_tile=tile, acov_all=every_lag if local.acov_all else None)


def _device(group=None):
    """Where collective buffers live: the current GPU for NCCL, host for gloo."""
    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")


def stop_sync(group=None):
    """The global stop rule for ``run_fsm_batched(..., stop_sync=...)``.

    Called once per run with this rank's (stop tick, all chains done, first
    failure key, failure record); returns the same fields for the whole
    batch: the max stop tick, whether every rank finished, and the smallest
    failure key (tick << 24 | global chain) with its owner's record
    (kind, label, sample index), so every rank raises the reference's first
    failure."""
    def sync(ticks: int, done: bool, err_key: int, err_rec: tuple) -> tuple:
        dev = _device(group)
        big = (1 << 62)
        t = torch.tensor([ticks, 0 if done else 1, -min(err_key, big)], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        g_ticks, any_undone, g_key = int(t[0]), bool(t[1]), -int(t[2])
        rec = torch.tensor(list(err_rec) if err_key == g_key < big else [0, 0, 0],
                           dtype=torch.int64, device=dev)
        dist.all_reduce(rec, op=dist.ReduceOp.SUM, group=group)
        return g_ticks, not any_undone, g_key, tuple(int(v) for v in rec)
    return sync


def _gather_cols(x, group):
    """Concatenate [rows, m_local] matrices of every rank along the chain axis
    (shards may differ in width by one)."""
    dev = _device(group)
    t = torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x).to(dev)
    t = t.to(torch.int64)
    w = torch.tensor([t.shape[1]], dtype=torch.int64, device=dev)
    world = dist.get_world_size(group)
    widths = [torch.zeros_like(w) for _ in range(world)]
    dist.all_gather(widths, w, group=group)
    widths = [int(v) for v in widths]
    mx = max(widths)
    pad = torch.zeros((t.shape[0], mx), dtype=torch.int64, device=dev)
    pad[:, :t.shape[1]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    return torch.cat([p[:, :wd] for p, wd in zip(parts, widths)], dim=1).cpu().numpy()


def global_ledger(ledger, group=None):
    """The whole batch's CostLedger from every rank's shard ledger (every rank
    gets it): count matrices gathered along the chain axis in rank order
    (= chain order, shard_range), block_exec_counts and native_shared_evals
    summed, tick_count and walltime the max, charged_cost re-derived from
    the global tick_count (lockstep.py:419-451)."""
    from .lockstep import CostLedger
    if not ledger.regime.startswith("fsm"):
        raise ValueError("global_ledger merges ledgers of FSM runs (run_fsm_batched); a sharded "
                         "lock-step charge needs the per-sample max over every rank's chains")
    dev = _device(group)
    blocks = torch.as_tensor(np.asarray(ledger.block_exec_counts if not isinstance(
        ledger.block_exec_counts, torch.Tensor) else ledger.block_exec_counts.cpu()),
        dtype=torch.int64).to(dev)
    dist.all_reduce(blocks, op=dist.ReduceOp.SUM, group=group)
    sc = torch.tensor([ledger.native_shared_evals], dtype=torch.int64, device=dev)
    dist.all_reduce(sc, op=dist.ReduceOp.SUM, group=group)
    mx = torch.tensor([float(ledger.tick_count), float(ledger.walltime)], dtype=torch.float64,
                      device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    ticks = int(mx[0])

    def host(x):
        return x.cpu() if isinstance(x, torch.Tensor) else x

    return CostLedger(
        iter_counts=_gather_cols(host(ledger.iter_counts), group),
        loop_exec_counts={s: _gather_cols(host(v), group) for s, v in ledger.loop_exec_counts.items()},
        tick_count=ticks, block_exec_counts=blocks.cpu().numpy(),
        charged_cost=ticks * ledger.tick_cost,
        walltime=float(mx[1]), regime=ledger.regime, tick_cost=ledger.tick_cost,
        shared_evals_per_tick=ledger.shared_evals_per_tick, native_shared_evals=int(sc.item()),
        sample_ticks=None if ledger.sample_ticks is None else _gather_cols(host(ledger.sample_ticks), group),
        extras=dict(ledger.extras))
