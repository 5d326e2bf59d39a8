"""Chain sharding across GPUs (one process per GPU, torch.distributed).

Chains are independent (``prng.py:84-94``): rank r of W owns the contiguous
chains [r*m/W, (r+1)*m/W) and runs them with no data-path collective.  At
the end, the diagnostics' partial moments are all-reduced (NCCL over NVLink
on GPUs, gloo in the CPU tests): chain-mean sums, the spread of chain means
(two-pass, no cancellation), max chain variance, and lag tiles of summed
autocovariances fetched only as far as Geyer's truncation needs.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .analysis import LAG_TILE, DiagMoments

__all__ = ["shard_range", "allreduce_moments", "LocalMoments"]


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
