"""Distributional parity harness: where a run is not
expected to be bit-identical to the reference (reduced-precision evaluators,
the fp32 throughput mode), two samplers must agree in distribution.

Unit of comparison: one post-burn-in chain mean per chain.  Chains are
independent (their streams are split from the seed, prng.py:84-94), so the
m chain means of a run are m iid draws of one law (a batch-means view that
needs no autocorrelation model), and two runs from different seeds give two
independent samples of it.  Per dimension:

* means: |mean_a - mean_b| <= z * sqrt(se_a^2 + se_b^2)  (Monte Carlo s.e.)
* spread: |log(var_a / var_b)| <= z * sqrt(2/(m_a-1) + 2/(m_b-1))
* two-sample Kolmogorov-Smirnov on the chain means: p > alpha / d

with z the two-sided normal quantile at alpha / d (Bonferroni over the d
dimensions: the family-wise false-alarm rate is alpha).
"""

import numpy as np


def compare_runs(a, b, burn, alpha=0.01):
    from scipy import stats
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    ca, cb = a[burn:].mean(axis=0), b[burn:].mean(axis=0)      # [m, d]
    ma, mb = ca.shape[0], cb.shape[0]
    d = ca.shape[1]
    z = float(stats.norm.isf(alpha / (2 * d)))
    se = np.sqrt(ca.var(axis=0, ddof=1) / ma + cb.var(axis=0, ddof=1) / mb)
    dm = np.abs(ca.mean(axis=0) - cb.mean(axis=0))
    lvr = np.abs(np.log(ca.var(axis=0, ddof=1) / cb.var(axis=0, ddof=1)))
    lvr_tol = z * np.sqrt(2.0 / (ma - 1) + 2.0 / (mb - 1))
    ks_p = np.array([stats.ks_2samp(ca[:, k], cb[:, k]).pvalue for k in range(d)])
    return {"d": d, "m": (ma, mb), "z": z,
            "max_mean_z": float(np.max(dm / se)),
            "max_logvar_ratio_over_tol": float(np.max(lvr / lvr_tol)),
            "min_ks_p": float(ks_p.min()), "ks_threshold": alpha / d,
            "ok_mean": bool(np.all(dm <= z * se)), "ok_var": bool(np.all(lvr <= lvr_tol)),
            "ok_ks": bool(np.all(ks_p > alpha / d))}


def assert_same_law(a, b, burn, alpha=0.01):
    r = compare_runs(a, b, burn, alpha)
    assert r["ok_mean"] and r["ok_var"] and r["ok_ks"], r
    return r
