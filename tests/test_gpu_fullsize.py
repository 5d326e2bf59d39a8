"""BASELINE.json configurations at their full chain counts, through the same
run options bench.py times (draw windows in 4 overlapped parts for C2, the
batched DTRMM prior in 3 parts for C4), checked with a size-independent
property: chain j's trajectory depends only on (seed, j, target)
(prng.py:84-94, lockstep.py:187), so every chain of the full-size run must
equal the oracle's run of that chain alone (chain_offset = j).  Step counts
bit-exact, samples within the tolerance of the smaller parity tests.  The C3
run also checks the pooled posterior moments against the closed form.
"""

import numpy as np
import pytest

from golden_cases import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fm():
    import paper_2503_17405_b200 as fm
    return fm


def _chain_ids(m):
    rng = np.random.default_rng(m)
    mid = np.sort(rng.choice(np.arange(4, m - 4), 4, replace=False))
    return [(0, 4), (m - 4, m)] + [(int(j), int(j) + 1) for j in mid]


def _full_run(fm, cfg, n, seed):
    import bench
    bundle, target = bench.make_workload(cfg, fm)
    batch = fm.init_batch(bundle, target, cfg["m"], seed)
    return fm.run_fsm_batched(bundle, target, batch, n, step_variant=cfg["variant"],
                              lanes=cfg.get("lanes", 0), draw_window=cfg.get("draw_window", 0),
                              draw_parts=cfg.get("draw_parts", 1),
                              prior_transform=cfg.get("prior_transform"),
                              prior_parts=cfg.get("prior_parts", 1))


@pytest.mark.parametrize("name,n,tol", [("c2", 100, 1e-11), ("c1", 200, 1e-11),
                                        ("c3", 50, 1e-11), ("c4", 10, 1e-10)])
def test_full_size_config_matches_oracle_per_chain(fm, name, n, tol):
    import bench
    from oracle import oracle as O
    cfg = bench.CONFIGS[name]
    seed = 11
    samples, led = _full_run(fm, cfg, n, seed)
    samples = np.asarray(samples)
    m = cfg["m"]
    assert samples.shape == (n, m, cfg["d"])
    assert np.isfinite(samples).all()
    assert (np.asarray(led.iter_counts) >= 0).all()
    okern, otarg = bench.make_workload(cfg, oracle=True)
    for lo, hi in _chain_ids(m):
        ref = O.run_fsm(okern, otarg, hi - lo, n, seed, variant=cfg["variant"],
                        chain_offset=lo, nthreads=8)
        assert np.array_equal(np.asarray(led.iter_counts)[:, lo:hi], ref["iter_counts"]), (lo, hi)
        assert rel_err(samples[:, lo:hi], ref["samples"]) <= tol, (lo, hi)


def test_full_size_c3_posterior_moments(fm):
    """C3 (16384 chains, equicorrelated Gaussian rho=0.99, zero mean, x0 = 0):
    the pooled mean of every coordinate lies within 6 Monte Carlo standard
    errors of 0, and the fast-mixing component x - mean(x) 1 (eigenvalue
    1 - rho) has the closed-form variance (1 - rho)(1 - 1/d) within 10%."""
    import bench
    cfg = bench.CONFIGS["c3"]
    d, rho = cfg["d"], 0.99
    samples, _ = _full_run(fm, cfg, 200, 3)
    s = np.asarray(samples)[50:]                      # burn-in
    chain_means = s.mean(axis=0)                      # [m, d]
    se = chain_means.std(axis=0, ddof=1) / np.sqrt(chain_means.shape[0])
    assert (np.abs(chain_means.mean(axis=0)) <= 6 * se + 1e-12).all()
    perp = s - s.mean(axis=-1, keepdims=True)
    var = perp.reshape(-1, d).var(axis=0)
    want = (1 - rho) * (1 - 1 / d)
    assert np.all(np.abs(var / want - 1) < 0.1), (var.min() / want, var.max() / want)
