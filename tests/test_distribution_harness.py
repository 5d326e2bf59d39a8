"""CPU checks of the distributional parity harness (tests/distribution_checks.py):
it accepts two independent samples of one law and rejects a shift of a few
Monte Carlo standard errors or a changed spread."""

import numpy as np

from distribution_checks import compare_runs


def _runs(shift=0.0, scale=1.0, seed=0, m=512, d=16, n=20):
    rng = np.random.default_rng(seed)
    a = rng.normal(size=(n, m, d))
    b = rng.normal(size=(n, m, d)) * scale + shift
    return a, b


def test_same_law_passes():
    oks = [compare_runs(*_runs(seed=s), burn=5) for s in range(20)]
    assert sum(r["ok_mean"] and r["ok_var"] and r["ok_ks"] for r in oks) >= 19


def test_mean_shift_is_detected():
    # chain means have sd 1/sqrt(15); a 0.06 shift is ~8 standard errors at m=512
    r = compare_runs(*_runs(shift=0.06), burn=5)
    assert not r["ok_mean"]


def test_spread_change_is_detected():
    r = compare_runs(*_runs(scale=1.5), burn=5)
    assert not r["ok_var"]
