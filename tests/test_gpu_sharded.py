"""Sharded runs (distributed.py) on one GPU: two gloo ranks, each owning a
contiguous chain shard (shard_range, init_batch(chain_offset=lo)), reproduce
the single-process run of the whole batch -- samples and every per-sample
count column by column, and, through stop_sync + global_ledger, the global
quantities the reference defines over all chains: tick_count (the chunked
stop rule, lockstep.py:359-366), the surplus-inclusive block_exec_counts and
native_shared_evals (lockstep.py:393-394, 419-451) and the first failure in
(tick, chain) order (lockstep.py:390-391).

The ranks share the device but never wait on each other inside a kernel:
the only cross-rank steps are the host-side reductions after each launch."""

import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name, fm):
    if name == "drmh":
        return (fm.drmh_kernel(100, 0.1), fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0]),
                1001, 60, "bundled")
    if name == "ess":
        return fm.elliptical_kernel(), fm.conjugate_target(100), 130, 40, "amortized"
    if name == "nuts":
        return fm.nuts_kernel(0.05, 10), fm.equicorrelated_gaussian_target(100, 0.99), 257, 30, "bundled"
    # fault injection: NaN once x[0] > 2.8 (test_errors_match_reference's target)
    return fm.drmh_kernel(5, 1.0), fm.targets.nan_band_target(2, 2.8, math.nan), 40, 400, "plain"


def _run(fm, name, lo, hi, stop_sync=None):
    bundle, target, m, n, variant = _case(name, fm)
    batch = fm.init_batch(bundle, target, hi - lo, 9, chain_offset=lo)
    try:
        s, led = fm.run_fsm_batched(bundle, target, batch, n, step_variant=variant,
                                    record_sample_ticks=True, stop_sync=stop_sync)
    except fm.KernelRunError as e:
        return ("error", e.chain, e.iteration, str(e.cause))
    return s, led


def worker(rank, world, port, name, q):
    import sys
    import traceback
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2503_17405_b200 as fm
        from paper_2503_17405_b200 import distributed
        m = _case(name, fm)[2]
        lo, hi = distributed.shard_range(m, rank, world)
        out = _run(fm, name, lo, hi, distributed.stop_sync())
        if isinstance(out[0], str):        # ("error", chain, iteration, cause)
            q.put((rank, out))
        else:
            s, led = out
            g = distributed.global_ledger(led)
            q.put((rank, (lo, hi, s, g.iter_counts, g.sample_ticks, g.tick_count,
                          np.asarray(g.block_exec_counts).tolist(), g.native_shared_evals,
                          led.tick_count)))
        dist.destroy_process_group()
    except BaseException:
        q.put((rank, ("exception", traceback.format_exc())))


def _spawn(name, world=2):
    import queue
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            rank, out = q.get(timeout=240)
            res[rank] = out
            if isinstance(out[0], str) and out[0] == "exception":   # the other rank may wait in a collective
                raise AssertionError(f"rank {rank} failed:\n{out[1]}")
    except queue.Empty:
        raise AssertionError(f"ranks {sorted(set(range(world)) - set(res))} sent nothing in 240 s")
    finally:
        for p in procs:
            p.join(60)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("name", ["drmh", "ess", "nuts"])
def test_two_shards_reproduce_the_whole_batch(name):
    import paper_2503_17405_b200 as fm
    m = _case(name, fm)[2]
    s, led = _run(fm, name, 0, m)
    res = _spawn(name)
    for rank, (lo, hi, s_r, it, st, ticks, blocks, shared, local_ticks) in sorted(res.items()):
        assert np.array_equal(s_r, s[:, lo:hi])
        assert np.array_equal(it, led.iter_counts)
        assert np.array_equal(st, led.sample_ticks)
        assert ticks == led.tick_count == local_ticks
        assert blocks == np.asarray(led.block_exec_counts).tolist()
        assert shared == led.native_shared_evals


def test_first_failure_is_raised_on_every_rank():
    import paper_2503_17405_b200 as fm
    whole = _run(fm, "nan", 0, 40)
    assert isinstance(whole[0], str) and whole[0] == "error"
    res = _spawn("nan")
    for rank, out in res.items():
        assert isinstance(out[0], str) and out[0] == "error"
        assert out[1:3] == whole[1:3], (rank, out, whole)
        assert out[3] == whole[3]
