"""World-size-2 gloo test of the multi-GPU diagnostics path (CPU): each rank
owns a contiguous chain shard (distributed.shard_range), computes its partial
moments, and allreduce_moments + ess_from_moments must give the same ESS /
R-hat as the single-process computation over all chains."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def local_moments(x, burn):
    """numpy partials of one shard [n, m_loc, d] (what diag_moments computes
    on a device): chain means, max chain variance, lag tiles of summed acov."""
    from paper_2503_17405_b200.analysis import LAG_TILE
    from paper_2503_17405_b200.distributed import LocalMoments
    y = x[burn:]
    n, m, d = y.shape
    means = y.mean(axis=0)
    c = y - means

    def tile(k):
        out = np.zeros((LAG_TILE, d))
        for t in range(LAG_TILE):
            lag = k * LAG_TILE + t
            if lag < n:
                out[t] = (c[: n - lag] * c[lag:]).sum(axis=(0, 1)) / n
        return out

    def every_lag():
        """sum over this shard's chains of every lag's autocovariance (by FFT,
        as diag_moments' acov_all does on the device)"""
        size = 1 << int(np.ceil(np.log2(2 * n)))
        f = np.fft.rfft(c, n=size, axis=0)
        return np.fft.irfft((f * np.conj(f)).sum(axis=1), n=size, axis=0)[:n].real / n

    return LocalMoments(n, means, y.var(axis=0).max(axis=0), tile, every_lag)


def global_moments(x, burn):
    from paper_2503_17405_b200.analysis import DiagMoments
    loc = local_moments(x, burn)
    m = x.shape[1]
    return DiagMoments(n=loc.n, m=m, d=x.shape[2], var_means=loc.chain_means.var(axis=0, ddof=1),
                       max_chain_var=loc.max_chain_var, acov_tile=loc.acov_tile)


def data():
    rng = np.random.default_rng(4)
    n, m, d = 300, 10, 3
    x = np.zeros((n, m, d))
    for i in range(1, n):
        x[i] = 0.9 * x[i - 1] + rng.normal(size=(m, d)) + 0.05 * np.arange(m)[:, None]
    return x


def worker(rank, world, port, q, every_lag=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_17405_b200 import analysis, distributed
    x = data()
    lo, hi = distributed.shard_range(x.shape[1], rank, world)
    loc = local_moments(x[:, lo:hi], 30)
    mom = distributed.allreduce_moments(loc)
    if every_lag:   # the all-lags path (C3/C5: slowly mixing chains) instead of lag tiles
        full = mom.acov_all() / mom.m
        ess = analysis._geyer_all(full, mom)[0]
        per = tuple(ess)
    else:
        per = analysis.ess_from_moments(mom).per_dimension
    rh = analysis.rhat_from_moments(mom)
    if rank == 0:
        q.put((per, tuple(rh)))
    dist.destroy_process_group()


def _spawn(target, world, *extra):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + extra) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    return [q.get(timeout=10) for _ in range(q.qsize() if hasattr(q, "qsize") else 1)]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_diagnostics_match_single_process():
    from paper_2503_17405_b200 import analysis
    (ess_dist, rh_dist), = _spawn(worker, 2)
    x = data()
    mom = global_moments(x, 30)
    ess = analysis.ess_from_moments(mom)
    assert np.allclose(ess_dist, ess.per_dimension, rtol=1e-12)
    assert np.allclose(rh_dist, analysis.rhat_from_moments(mom), rtol=1e-12)
    # and both agree with the reference formula on the raw chains
    from ess_reference import ess_numpy
    for k in range(x.shape[2]):
        assert ess.per_dimension[k] == pytest.approx(ess_numpy(x[30:, :, k].T), rel=1e-9)


def test_shard_ranges_partition_the_chains():
    from paper_2503_17405_b200.distributed import shard_range
    for m, w in ((10, 3), (1 << 20, 8), (7, 7)):
        spans = [shard_range(m, r, w) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_sharded_every_lag_path_matches_single_process():
    """acov_all (one transform over every lag, the path C3/C5 take) all-reduced
    over two ranks equals the single-process all-lags sums."""
    from paper_2503_17405_b200 import analysis
    (ess_dist, rh_dist), = _spawn(worker, 2, True)
    x = data()
    loc = local_moments(x, 30)
    mom = global_moments(x, 30)
    ess = analysis._geyer_all(loc.acov_all() / x.shape[1], mom)[0]
    assert np.allclose(ess_dist, ess, rtol=1e-10)
    from ess_reference import ess_numpy
    for k in range(x.shape[2]):
        assert ess[k] == pytest.approx(ess_numpy(x[30:, :, k].T), rel=1e-9)


def _oracle_full():
    from oracle import oracle as O
    return O.run_fsm(O.drmh(30, 0.5), O.mog(10, 0.9, [-3.0, 0.0, 3.0]), 9, 40, 3,
                     variant="bundled", nthreads=2)


def ledger_worker(rank, world, port, q):
    """Each rank holds its shard's columns of a real (oracle) ledger; the merged
    ledger must be the full one.  Then the stop rule: the max stop tick, the
    completion flag and the smallest failure key with its owner's record."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_17405_b200 import distributed
    from paper_2503_17405_b200.lockstep import CostLedger
    full = _oracle_full()
    lo, hi = distributed.shard_range(9, rank, world)
    blocks = np.array([rank + 1, 10 * (rank + 1), 100 * (rank + 1)], dtype=np.int64)
    led = CostLedger(iter_counts=full["iter_counts"][:, lo:hi],
                     loop_exec_counts={2: full["iter_counts"][:, lo:hi]},
                     tick_count=500 + 100 * rank, block_exec_counts=blocks, charged_cost=0.0,
                     walltime=1.0 + rank, regime="fsm-bundled", tick_cost=2.0,
                     native_shared_evals=7 * (rank + 1), sample_ticks=full["sample_ticks"][:, lo:hi])
    g = distributed.global_ledger(led)
    sync = distributed.stop_sync()
    big = 1 << 62
    key = ((450 << 24) | 7) if rank == 1 else big
    s1 = sync(500 + 100 * rank, True, key, (1, 2, 3) if rank == 1 else (0, 0, 0))
    s2 = sync(300, rank == 0, big, (0, 0, 0))
    q.put((rank, g.iter_counts, g.loop_exec_counts[2], g.sample_ticks, g.block_exec_counts.tolist(),
           g.native_shared_evals, g.tick_count, g.walltime, g.charged_cost, s1, s2))
    dist.destroy_process_group()


def test_global_ledger_and_stop_rule_over_two_ranks():
    outs = _spawn(ledger_worker, 2)
    full = _oracle_full()
    assert len(outs) == 2
    for (rank, it, lx, st, blocks, shared, ticks, wall, charged, s1, s2) in outs:
        assert np.array_equal(it, full["iter_counts"]) and np.array_equal(lx, full["iter_counts"])
        assert np.array_equal(st, full["sample_ticks"])
        assert blocks == [3, 30, 300] and shared == 21
        assert ticks == 600 and wall == 2.0 and charged == 1200.0
        assert s1 == (600, True, (450 << 24) | 7, (1, 2, 3))
        assert s2[0] == 300 and s2[1] is False and s2[2] == 1 << 62
