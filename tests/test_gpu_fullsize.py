"""BASELINE.json configurations at their full chain counts AND the sample
horizons bench.py times (C1 n=1000, C2 n=1000, C3 n=1000, C4 n=200), through
the same run options (C2: draw windows in 4 overlapped parts; C4: the batched
DTRMM-class prior transform in 3 parts).

Chain j's trajectory depends only on (seed, j, target) (prng.py:84-94,
lockstep.py:187), so every chain of the full-size run can be replayed alone
by the oracle (chain_offset = j).  128 chains are checked per config: the
first 8, the last 8 and 112 spread at random.  Per chain the report gives the
first sample whose step count (iter_counts) or tick stamp (sample_ticks)
differs from the oracle's, and the largest relative sample difference before
it.  The parity contract: step counts bit-exact over the
horizon, samples within tolerance; where a floating-point ulp flips a branch
(a reduction order or a CUDA transcendental that differs from glibc by an
ulp), the chain's later trajectory is a different valid draw and parity is
distributional beyond that point (test_gpu_distribution.py).

`python tests/test_gpu_fullsize.py c3` prints the report as JSON.
"""

import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from golden_cases import rel_err  # noqa: E402

pytestmark = pytest.mark.gpu

# (config, horizon n = bench.py's, sample tolerance before divergence, minimum
# fraction of checked chains bit-exact over the whole horizon)
# (measured on B200, seed 11, 64 chains: every chain bit-exact over the whole
# horizon in all four configs; max relative sample error C1 2.2e-15, C2 0,
# C3 3.5e-13, C4 2.1e-15 -- profiles/r04_horizon_*.json)
HORIZONS = {"c1": (1000, 1e-12, 1.0), "c2": (1000, 1e-12, 1.0), "c3": (1000, 1e-11, 1.0),
            "c4": (200, 1e-12, 1.0)}


@pytest.fixture(scope="module")
def fm():
    import paper_2503_17405_b200 as fm
    return fm


def checked_chains(m, k=64):
    rng = np.random.default_rng(m)
    mid = np.sort(rng.choice(np.arange(8, m - 8), k - 16, replace=False)) if m > k else \
        np.arange(8, m - 8)
    return list(range(8)) + [int(j) for j in mid] + list(range(m - 8, m))


def _full_run(fm, cfg, n, seed):
    import bench
    bundle, target = bench.make_workload(cfg, fm)
    batch = fm.init_batch(bundle, target, cfg["m"], seed)
    return fm.run_fsm_batched(bundle, target, batch, n, step_variant=cfg["variant"],
                              record_sample_ticks=True, lanes=cfg.get("lanes", 0),
                              draw_window=cfg.get("draw_window", 0),
                              draw_parts=cfg.get("draw_parts", 1),
                              prior_transform=cfg.get("prior_transform"),
                              prior_parts=cfg.get("prior_parts", 1), surplus=False,
                              output="torch")


def horizon_report(fm, name, n=None, seed=11, k=128):
    """Full-size device run of config `name` against the oracle, chain by chain."""
    import bench
    from oracle import oracle as O
    cfg = bench.CONFIGS[name]
    n = n or HORIZONS[name][0]
    samples, led = _full_run(fm, cfg, n, seed)
    m = cfg["m"]
    chains = checked_chains(m, k)
    finite = bool(samples.isfinite().all())
    idx = __import__("torch").as_tensor(chains, device=samples.device)
    sel = samples.index_select(1, idx).cpu().numpy()          # [n, k, d]: only the checked chains
    its = led.iter_counts.index_select(1, idx.to(led.iter_counts.device)).cpu().numpy()
    ticks = led.sample_ticks.index_select(1, idx.to(led.sample_ticks.device)).cpu().numpy()
    del samples
    okern, otarg = bench.make_workload(cfg, oracle=True)

    def one(j):
        return j, O.run_fsm(okern, otarg, 1, n, seed, variant=cfg["variant"], chain_offset=j)

    with ThreadPoolExecutor(os.cpu_count() or 4) as pool:
        refs = dict(pool.map(one, chains))
    rows = []
    for c, j in enumerate(chains):
        r = refs[j]
        diff = (its[:, c] != r["iter_counts"][:, 0]) | (ticks[:, c] != r["sample_ticks"][:, 0])
        first = int(np.argmax(diff)) if diff.any() else n
        err = rel_err(sel[:first, c], r["samples"][:first, 0])
        rows.append({"chain": j, "first_divergent_sample": first if first < n else None,
                     "max_rel_err_before": err})
    exact = [r for r in rows if r["first_divergent_sample"] is None]
    firsts = [r["first_divergent_sample"] for r in rows if r["first_divergent_sample"] is not None]
    return {"config": name, "workload": cfg["workload"], "m": m, "n": n, "seed": seed,
            "chains_checked": len(rows), "bit_exact_chains": len(exact),
            "bit_exact_fraction": len(exact) / len(rows),
            "earliest_divergence": min(firsts) if firsts else None,
            "max_rel_err_before_divergence": max(r["max_rel_err_before"] for r in rows),
            "finite": finite, "chains": rows}


@pytest.mark.parametrize("name", sorted(HORIZONS))
def test_full_size_config_matches_oracle_at_bench_horizon(fm, name):
    n, tol, min_frac = HORIZONS[name]
    rep = horizon_report(fm, name)
    out = os.environ.get("FSMC_HORIZON_OUT")
    if out:
        with open(os.path.join(out, f"horizon_{name}.json"), "w") as f:
            json.dump(rep, f, indent=1)
    print(f"\n{name}: {rep['bit_exact_chains']}/{rep['chains_checked']} chains bit-exact over "
          f"n={n}; earliest divergence {rep['earliest_divergence']}; max rel err before "
          f"divergence {rep['max_rel_err_before_divergence']:.2e}")
    assert rep["finite"]
    assert rep["max_rel_err_before_divergence"] <= tol
    assert rep["bit_exact_fraction"] >= min_frac


def test_full_size_c3_posterior_moments(fm):
    """C3 (16384 chains, equicorrelated Gaussian rho=0.99, zero mean, x0 = 0):
    the pooled mean of every coordinate lies within 6 Monte Carlo standard
    errors of 0, and the fast-mixing component x - mean(x) 1 (eigenvalue
    1 - rho) has the closed-form variance (1 - rho)(1 - 1/d) within 10%."""
    import bench
    cfg = bench.CONFIGS["c3"]
    d, rho = cfg["d"], 0.99
    samples, _ = _full_run(fm, cfg, 200, 3)
    s = samples[50:].cpu().numpy()                    # burn-in
    chain_means = s.mean(axis=0)                      # [m, d]
    se = chain_means.std(axis=0, ddof=1) / np.sqrt(chain_means.shape[0])
    assert (np.abs(chain_means.mean(axis=0)) <= 6 * se + 1e-12).all()
    perp = s - s.mean(axis=-1, keepdims=True)
    var = perp.reshape(-1, d).var(axis=0)
    want = (1 - rho) * (1 - 1 / d)
    assert np.all(np.abs(var / want - 1) < 0.1), (var.min() / want, var.max() / want)


if __name__ == "__main__":
    import paper_2503_17405_b200 as _fm
    for nm in sys.argv[1:] or sorted(HORIZONS):
        r = horizon_report(_fm, nm)
        r.pop("chains") if os.environ.get("BRIEF") else None
        print(json.dumps(r))
