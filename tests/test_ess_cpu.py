"""CPU checks of the ESS diagnostics' host half: the dimension-vectorized
Geyer truncation (analysis._geyer_all, used by effective_sample_size) against
the per-dimension restatement (analysis._ess_dim) bit for bit, and against
the reference formula (tests/ess_reference.py) on real draws."""

import warnings

import numpy as np
import pytest

from paper_2503_17405_b200 import analysis as A


def _moments(acf_sum, n, m, var_means, max_chain_var):
    d = acf_sum.shape[1]
    pad = np.vstack([acf_sum, np.zeros((A.LAG_TILE, d))])
    return A.DiagMoments(n=n, m=m, d=d, var_means=var_means, max_chain_var=max_chain_var,
                         acov_tile=lambda k: pad[A.LAG_TILE * k: A.LAG_TILE * (k + 1)],
                         acov_all=lambda: acf_sum)


def test_vectorized_geyer_equals_per_dimension_restatement():
    rng = np.random.default_rng(0)
    warnings.simplefilter("ignore")
    for _ in range(600):
        n, m, d = int(rng.integers(10, 300)), int(rng.integers(1, 6)), int(rng.integers(1, 6))
        phi = rng.uniform(-0.9, 0.999, size=d)
        t = np.arange(n)[:, None]
        acf = (phi[None, :] ** t) * rng.uniform(0.5, 2, size=d) + rng.normal(0, 0.02, size=(n, d))
        vm = rng.uniform(0, 0.5, size=d) if m > 1 else np.zeros(d)
        mcv = np.where(rng.uniform(size=d) < 0.05, 0.0, 1.0)
        mom = _moments(acf * m, n, m, vm, mcv)
        ac = A._Acov(mom)
        ref = [A._ess_dim(ac, mom, k) for k in range(d)]
        got = A.ess_from_moments(mom)
        assert list(got.per_dimension) == [e for e, _ in ref]
        assert got.flagged == any(f for _, f in ref)


@pytest.mark.parametrize("phi", [0.0, 0.5, 0.95, -0.6])
def test_ess_matches_reference_formula_on_draws(phi):
    from ess_reference import ess_numpy
    rng = np.random.default_rng(3)
    n, m, d = 400, 6, 3
    x = np.zeros((n, m, d))
    e = rng.normal(size=(n, m, d))
    for i in range(1, n):
        x[i] = phi * x[i - 1] + e[i]
    size = 2 ** int(np.ceil(np.log2(2 * n)))
    cen = x - x.mean(axis=0, keepdims=True)
    f = np.fft.rfft(cen, n=size, axis=0)
    acov = np.fft.irfft(f * np.conj(f), n=size, axis=0)[:n].real / n       # [n, m, d]
    mom = _moments(acov.sum(axis=1), n, m, x.mean(axis=0).var(axis=0, ddof=1),
                   x.var(axis=0).max(axis=0))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        got = A.ess_from_moments(mom).per_dimension
        ref = [ess_numpy(x[:, :, k].T) for k in range(d)]
    np.testing.assert_allclose(got, ref, rtol=1e-10)


def test_vectorized_geyer_stops_at_nan_pair_like_the_reference_loop():
    """The reference's truncation loop runs `while ... and pair_sum >= 0`
    (analysis.py:353-374), so a NaN pair sum ends it exactly as a negative one
    does; the vectorized form must agree (including a NaN in pair 0)."""
    rng = np.random.default_rng(5)
    warnings.simplefilter("ignore")
    for case in range(200):
        n, m, d = int(rng.integers(20, 200)), int(rng.integers(2, 5)), int(rng.integers(1, 5))
        phi = rng.uniform(0.3, 0.99, size=d)
        acf = (phi[None, :] ** np.arange(n)[:, None]) * rng.uniform(0.5, 2, size=d)
        for k in range(d):
            at = int(rng.integers(1, min(n, 40)))
            acf[at, k] = np.nan
        mom = _moments(acf * m, n, m, rng.uniform(0, 0.5, size=d), np.ones(d))
        ac = A._Acov(mom)
        ref = [A._ess_dim(ac, mom, k) for k in range(d)]
        ess, bad, _ = A._geyer_all(A._acf_for_geyer(mom), mom)
        got = [A.ess_from_moments(mom).per_dimension[k] for k in range(d)]
        assert got == [e for e, _ in ref], case
