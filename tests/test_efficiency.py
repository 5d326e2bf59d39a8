"""Cost-theory analytics (paper_2503_17405_b200.efficiency) against values
frozen from the live reference (tests/golden/efficiency.npz, analysis.py:53-324)
and the reference's own analytic anchors (pkg/tests/test_analysis.py:23-120).
Host only: numpy inputs, plus torch CPU tensors standing in for device ledgers."""

import math

import numpy as np
import pytest
import torch

from golden_cases import load
from paper_2503_17405_b200 import analysis as A
from paper_2503_17405_b200.lockstep import CostParams

PARAMS = CostParams(block_costs=(0.05, 1.0, 0.05), alpha=1.0, loop_states=(2,))


def test_costs_and_report_match_reference():
    g = load("efficiency")
    N = g["N"]
    for src in (N, torch.as_tensor(N, dtype=torch.int32)):
        assert A.barrier_cost(src) == float(g["barrier"])
        assert A.desync_cost(src) == float(g["desync"])
        rep = A.efficiency_report(PARAMS, src, standard_cost_per_sample=3.0, fsm_cost_per_sample=1.5)
        got = np.array([rep.m, rep.E_of_m, rep.R_of_m, rep.mean_N, rep.mean_max_N])
        np.testing.assert_allclose(got, g["report"], rtol=1e-13)


def test_bound_R_monte_carlo_reproduces_reference_draws():
    g = load("efficiency")
    flat = g["N"].reshape(-1)
    for m in (1, 16, 1024):
        b = A.bound_R(m, samples=flat, n_replicates=2000, seed=5)
        np.testing.assert_allclose([b.estimate, b.std_error], g[f"bound_{m}"], rtol=1e-12)
    b = A.bound_R(16, bernoulli=(0.1, 3.0), n_replicates=20_000, seed=1)
    np.testing.assert_allclose([b.estimate, b.std_error, b.closed_form], g["bound_bern"], rtol=1e-12)


def test_bound_R_exact_agrees_with_monte_carlo_within_its_error():
    """method='exact' is the limit the reference's estimator converges to."""
    g = load("efficiency")
    flat = g["N"].reshape(-1)
    for m in (1, 16, 1024):
        ex = A.bound_R(m, samples=torch.as_tensor(flat), n_replicates=2000, method="exact")
        mc = g[f"bound_{m}"]
        assert abs(ex.estimate - mc[0]) <= 5 * max(mc[1], 1e-12) + 1e-12, m
        if m > 1:
            assert ex.std_error == pytest.approx(mc[1], rel=0.2)
    assert A.bound_R(1, samples=flat, method="exact").estimate == pytest.approx(1.0, abs=1e-12)
    ex = A.bound_R(16, bernoulli=(0.1, 3.0), method="exact")
    assert ex.estimate == ex.closed_form == A.bernoulli_bound_closed_form(0.1, 16)
    # two-point law of pkg/tests/test_analysis.py:61-67, exactly
    ex = A.bound_R(4, samples=np.array([0, 0, 0, 10.0]), method="exact")
    assert ex.estimate == pytest.approx((1 - 0.75 ** 4) / 0.25, rel=1e-14)
    # m in the tens of thousands (BASELINE config 2) needs no resampling
    big = A.bound_R(65536, samples=flat, method="exact")
    assert 1.0 < big.estimate <= flat.max() / flat.mean() + 1e-12


def test_prop_bound_and_concentration_match_reference():
    g = load("efficiency")
    rep = A.verify_prop_bound(500, seed=3)
    ref = g["prop"]
    assert len(rep.violations) == int(ref[0]) == 0
    assert rep.tightness_cases == int(ref[1])
    assert rep.tightness_max_rel_err < 1e-12
    runs = list(g["conc_runs"])
    c = A.concentration_check(runs, (10, 100, 1000, 4000), PARAMS)
    got = np.array([c.slope, c.slope_stderr, c.limit_estimate, *c.deviations])
    np.testing.assert_allclose(got, g["conc"], rtol=1e-9)
    ct = A.concentration_check([torch.as_tensor(r) for r in runs], (10, 100, 1000, 4000), PARAMS)
    assert ct.slope == pytest.approx(c.slope, rel=1e-12)


def test_reference_anchors():
    """pkg/tests/test_analysis.py:23-120 restated."""
    p3 = CostParams(block_costs=(1.0, 1.0, 1.0), alpha=1.0, loop_states=(2,))
    assert A.efficiency_model(p3, 6.0, 18.0) == pytest.approx(20.0 / 24.0)
    assert A.efficiency_model(CostParams(block_costs=(1.0,), alpha=1.0), 6.0, 18.0) == \
        pytest.approx(3.0)
    with pytest.raises(ValueError):
        A.efficiency_model(CostParams(block_costs=(1.0, 1.0, 1.0), loop_states=(2, 3)), 2.0, 3.0)
    with pytest.raises(ValueError):
        A.efficiency_model(CostParams(block_costs=(1.0,)), 0.0, 1.0)
    assert A.bernoulli_bound_closed_form(0.5, 2) == pytest.approx(1.5, abs=1e-15)
    with pytest.raises(ValueError):
        A.bound_R(2)
    with pytest.raises(ValueError):
        A.bound_R(2, samples=np.array([]))
    with pytest.raises(ValueError):
        A.bound_R(0, bernoulli=(0.5, 1.0))
    runs = [np.full((1000, 4), 3, dtype=np.int64) for _ in range(5)]
    rep = A.concentration_check(runs, (10, 100, 500, 1000), p3)
    assert rep.degenerate and rep.slope is None
    rng = np.random.default_rng(4)
    runs = [rng.geometric(0.4, size=(20_000, 4)) for _ in range(16)]
    rep = A.concentration_check(runs, (20, 200, 2000, 20_000),
                                CostParams(block_costs=(0.0, 1.0, 0.0), alpha=1.0, loop_states=(2,)))
    assert -0.65 < rep.slope < -0.35
    assert A.hoeffding_rate(500, 0.05) / A.hoeffding_rate(1000, 0.05) == pytest.approx(math.sqrt(2))
    with pytest.raises(ValueError):
        A.efficiency_report(p3, np.zeros((3, 2)) + 1.0, 1.0, 1.0).__class__(
            m=1, E_of_m=1.0, R_of_m=0.5, mean_N=1.0, mean_max_N=1.0,
            standard_cost_per_sample=1.0, fsm_cost_per_sample=1.0)
