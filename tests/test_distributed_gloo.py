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

    return LocalMoments(n, means, y.var(axis=0).max(axis=0), tile)


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


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_17405_b200 import analysis, distributed
    x = data()
    lo, hi = distributed.shard_range(x.shape[1], rank, world)
    mom = distributed.allreduce_moments(local_moments(x[:, lo:hi], 30))
    ess = analysis.ess_from_moments(mom)
    rh = analysis.rhat_from_moments(mom)
    if rank == 0:
        q.put((ess.per_dimension, tuple(rh)))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_diagnostics_match_single_process():
    from paper_2503_17405_b200 import analysis
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ess_dist, rh_dist = q.get(timeout=10)
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
