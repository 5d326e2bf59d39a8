"""Cost theory over the device ledgers (drop-in for ``fsm_mcmc.analysis``'s
efficiency half, ``analysis.py:53-324``).

Everything here is arithmetic over the inner-loop counts N[i, j] (chain j's
loop executions for its i-th sample) that ``run_fsm_batched`` /
``run_standard_batched`` return.  With ``output="torch"`` those stay in HBM
as int32 tensors; the reductions below (row maxima, column sums, means) then
run on the device and only scalars cross to the host.  numpy inputs are
reduced on the host exactly as before.

``bound_R`` keeps the reference's Monte-Carlo estimator (same numpy
generator, so the same seed gives the same draws) and adds
``method="exact"``: for integer counts the bootstrap expectation it
estimates, E[max of m draws from the empirical law], is a finite sum over
the empirical CDF, E[max] = sum_t (1 - F(t)^m), with no resampling at all.
That is what makes R(m) at m = 65536 chains (BASELINE config 2) instant.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .lockstep import CostParams

__all__ = ["barrier_cost", "desync_cost", "efficiency_model", "efficiency_report",
           "EfficiencyReport", "bound_R", "BoundEstimate", "bernoulli_bound_closed_form",
           "verify_prop_bound", "PropBoundReport", "concentration_check", "ConcentrationReport",
           "hoeffding_rate", "empirical_max_moments"]


def _counts(N):
    """(n, m) count matrix as a float64 tensor on its own device, or numpy."""
    if isinstance(N, torch.Tensor):
        return N.to(torch.float64)
    return np.asarray(N, dtype=float)


def barrier_cost(iter_counts) -> float:
    """sum_i max_j N_ij: every iteration waits for the slowest chain (analysis.py:53-56)."""
    N = _counts(iter_counts)
    if isinstance(N, torch.Tensor):
        return float(N.max(dim=1).values.sum().item())
    return float(N.max(axis=1).sum())


def desync_cost(iter_counts) -> float:
    """max_j sum_i N_ij: chains run free of barriers (analysis.py:59-62)."""
    N = _counts(iter_counts)
    if isinstance(N, torch.Tensor):
        return float(N.sum(dim=0).max().item())
    return float(N.sum(axis=0).max())


def _loop_state(params: CostParams, loop_state):
    """The single loop state the E(m) model prices (analysis.py:65-74)."""
    if loop_state is not None:
        return loop_state
    if len(params.block_costs) == 1:
        return 1
    if len(params.loop_states) == 1:
        return params.loop_states[0]
    raise ValueError("efficiency_model needs a unique loop state; pass loop_state explicitly")


def efficiency_model(params: CostParams, mean_N: float, mean_max_N: float,
                     loop_state: int | None = None) -> float:
    """E(m) = (c_rest + c_loop E[max_j N_j]) / (alpha (c_rest + c_loop) (K - 1 + E[N]))
    (analysis.py:77-95; Prop. 1)."""
    if mean_N <= 0:
        raise ValueError(f"mean_N must be positive, got {mean_N}")
    costs = params.full_block_costs()
    c_loop = costs[_loop_state(params, loop_state) - 1]
    c_rest = sum(costs) - c_loop
    denom = params.alpha * (c_rest + c_loop) * (len(costs) - 1 + mean_N)
    if denom == 0:
        raise ValueError("zero denominator: total block cost or mean_N degenerate")
    return (c_rest + c_loop * mean_max_N) / denom


@dataclass(frozen=True)
class EfficiencyReport:
    """Model efficiency of one paired run at m chains (analysis.py:98-111)."""

    m: int
    E_of_m: float
    R_of_m: float
    mean_N: float
    mean_max_N: float
    standard_cost_per_sample: float
    fsm_cost_per_sample: float

    def __post_init__(self):
        if self.R_of_m < 1.0 - 1e-9:
            raise ValueError(f"R(m) must be >= 1, got {self.R_of_m}")


def efficiency_report(params: CostParams, iter_counts, standard_cost_per_sample: float,
                      fsm_cost_per_sample: float, loop_state: int | None = None
                      ) -> EfficiencyReport:
    """Summary of a paired run from its N matrix and the two charged costs
    (analysis.py:114-130).  A device N is reduced on the device."""
    N = _counts(iter_counts)
    n, m = N.shape
    if isinstance(N, torch.Tensor):
        mean_N = float(N.mean().item())
        mean_max = float(N.max(dim=1).values.mean().item())
    else:
        mean_N = float(N.mean())
        mean_max = float(N.max(axis=1).mean())
    return EfficiencyReport(m=int(m), E_of_m=efficiency_model(params, mean_N, mean_max, loop_state),
                            R_of_m=mean_max / mean_N if mean_N > 0 else 1.0, mean_N=mean_N,
                            mean_max_N=mean_max, standard_cost_per_sample=standard_cost_per_sample,
                            fsm_cost_per_sample=fsm_cost_per_sample)


def bernoulli_bound_closed_form(p: float, m: int) -> float:
    """R(m) when N/B ~ Bernoulli(p): (1 - (1 - p)^m) / p (analysis.py:133-140)."""
    if not 0 < p <= 1:
        raise ValueError(f"p must be in (0, 1], got {p}")
    if m < 1:
        raise ValueError(f"m must be >= 1, got {m}")
    return (1.0 - (1.0 - p) ** m) / p


@dataclass(frozen=True)
class BoundEstimate:
    m: int
    estimate: float
    std_error: float
    closed_form: float | None = None


def empirical_max_moments(values, probs, m: int) -> tuple[float, float, float]:
    """(E[N], E[M], E[M^2]) for M = max of m iid draws of a law on the
    nonnegative integers ``values`` with probabilities ``probs``.

    P(M <= t) = F(t)^m, so E[M] = sum_{t>=0} (1 - F(t)^m) and
    E[M^2] = sum_{t>=0} (2t + 1)(1 - F(t)^m).  (F^m is formed as
    exp(m log F) so m in the millions stays accurate.)"""
    values = np.asarray(values, dtype=np.int64)
    probs = np.asarray(probs, dtype=float)
    top = int(values.max())
    pmf = np.zeros(top + 1)
    np.add.at(pmf, values, probs)
    cdf = np.minimum(np.cumsum(pmf), 1.0)[:-1]              # F(0) .. F(top - 1)
    with np.errstate(divide="ignore"):
        tail = -np.expm1(m * np.log(cdf))                    # 1 - F(t)^m
    t = np.arange(top, dtype=float)
    return float(values @ probs), float(tail.sum()), float(((2.0 * t + 1.0) * tail).sum())


def bound_R(m: int, samples=None, bernoulli: tuple | None = None, n_replicates: int = 100_000,
            seed: int = 0, method: str = "mc") -> BoundEstimate:
    """R(m) = E[max of m iid N] / E[N] (analysis.py:150-186).

    ``method="mc"`` is the reference estimator (numpy ``default_rng(seed)``,
    ``n_replicates`` resampled maxima; same seed, same draws).
    ``method="exact"`` evaluates the expectation that estimator targets in
    closed form (integer counts; ``samples`` may be a device tensor) and
    reports the standard error ``n_replicates`` Monte-Carlo draws would have.
    """
    if m < 1:
        raise ValueError(f"m must be >= 1, got {m}")
    if (samples is None) == (bernoulli is None):
        raise ValueError("pass exactly one of samples= or bernoulli=")
    if method not in ("mc", "exact"):
        raise ValueError("method must be 'mc' or 'exact'")
    closed = None
    if bernoulli is not None:
        p, B = bernoulli
        closed = bernoulli_bound_closed_form(p, m)
        mean_N = p * B
        if method == "exact":
            q = 1.0 - (1.0 - p) ** m                          # P(max = B)
            return BoundEstimate(m=m, estimate=closed, closed_form=closed,
                                 std_error=B * math.sqrt(q * (1.0 - q)) /
                                 math.sqrt(n_replicates) / mean_N)
        rng = np.random.default_rng(seed)
        maxima = (rng.random((n_replicates, m)) < p).any(axis=1).astype(float) * B
    else:
        if isinstance(samples, torch.Tensor):
            vals_t = samples.reshape(-1)
            if vals_t.numel() == 0:
                raise ValueError("empty sample")
            if bool((vals_t < 0).any()):
                raise ValueError("iteration counts must be nonnegative")
            if method == "exact":
                uniq, cnt = torch.unique(vals_t.to(torch.int64), return_counts=True)
                values, probs = uniq.cpu().numpy(), cnt.cpu().numpy() / float(vals_t.numel())
            else:
                vals = vals_t.to(torch.float64).cpu().numpy()
        else:
            vals = np.asarray(samples, dtype=float)
            if vals.size == 0:
                raise ValueError("empty sample")
            if np.any(vals < 0):
                raise ValueError("iteration counts must be nonnegative")
            if method == "exact":
                if not np.array_equal(vals, np.round(vals)):
                    raise ValueError("method='exact' needs integer iteration counts")
                values, cnt = np.unique(vals.astype(np.int64), return_counts=True)
                probs = cnt / float(vals.size)
        if method == "exact":
            mean_N, e_max, e_max2 = empirical_max_moments(values, probs, m)
            if mean_N <= 0:
                raise ValueError("sample mean must be positive")
            sd = math.sqrt(max(e_max2 - e_max * e_max, 0.0))
            return BoundEstimate(m=m, estimate=e_max / mean_N,
                                 std_error=sd / math.sqrt(n_replicates) / mean_N)
        mean_N = float(vals.mean())
        if mean_N <= 0:
            raise ValueError("sample mean must be positive")
        rng = np.random.default_rng(seed)
        maxima = vals[rng.integers(0, vals.size, size=(n_replicates, m))].max(axis=1)
    return BoundEstimate(m=m, estimate=float(maxima.mean()) / mean_N,
                         std_error=float(maxima.std(ddof=1)) / math.sqrt(n_replicates) / mean_N,
                         closed_form=closed)


@dataclass
class PropBoundReport:
    trials: int
    violations: list = field(default_factory=list)
    max_excess: float = 0.0
    tightness_cases: int = 0
    tightness_max_rel_err: float = 0.0

    @property
    def ok(self) -> bool:
        return not self.violations


def verify_prop_bound(trials: int, seed: int = 0, tol: float = 1e-12) -> PropBoundReport:
    """Random instances of E(m) <= R(m), with equality when K = 1 (analysis.py:215-260).

    Per trial: K in 1..6 block costs, an admissible alpha (its lower end with
    probability 1/4), m in 1..64, a bounded integer law for N with positive
    mean; both sides exact (``empirical_max_moments``).  The draw sequence
    follows the reference's, so a seed names the same instances."""
    if trials < 1:
        raise ValueError("trials must be >= 1")
    rng = np.random.default_rng(seed)
    rep = PropBoundReport(trials=trials)
    for t in range(trials):
        K = int(rng.integers(1, 7))
        m = int(rng.integers(1, 65))
        if K == 1:
            costs, alpha, k = (float(rng.uniform(0.1, 3.0)),), 1.0, 1
        else:
            costs = tuple(rng.uniform(0.0, 3.0, size=K))
            if sum(costs) == 0.0:
                costs = tuple(c + 0.1 for c in costs)
            k = int(rng.integers(1, K + 1))
            lo = max(costs) / sum(costs)
            alpha = lo if rng.random() < 0.25 else float(rng.uniform(lo, 1.0))
        B = int(rng.integers(1, 41))
        probs = rng.dirichlet(np.ones(B + 1))
        if probs[0] > 1.0 - 1e-9:
            probs = np.full(B + 1, 1.0 / (B + 1))
        mean_N, mean_max, _ = empirical_max_moments(np.arange(B + 1), probs, m)
        e_m = efficiency_model(CostParams(block_costs=costs, alpha=alpha, loop_states=(k,)),
                               mean_N, mean_max, loop_state=k)
        r_m = mean_max / mean_N
        if e_m > r_m + tol * max(1.0, abs(r_m)):
            rep.violations.append({"trial": t, "K": K, "m": m, "alpha": alpha, "costs": costs,
                                   "E": e_m, "R": r_m})
            rep.max_excess = max(rep.max_excess, e_m - r_m)
        if K == 1:
            rep.tightness_cases += 1
            rep.tightness_max_rel_err = max(rep.tightness_max_rel_err,
                                            abs(e_m - r_m) / max(abs(r_m), 1e-300))
    return rep


def hoeffding_rate(n: int, delta: float, scale: float = 1.0) -> float:
    """scale * ln(2/delta) / sqrt(n) (analysis.py:263-268)."""
    if n < 1 or not 0 < delta < 1:
        raise ValueError("need n >= 1 and delta in (0, 1)")
    return scale * math.log(2.0 / delta) / math.sqrt(n)


@dataclass(frozen=True)
class ConcentrationReport:
    n_grid: tuple
    deviations: tuple
    slope: float | None
    slope_stderr: float | None
    slope_ci95: tuple | None
    limit_estimate: float
    degenerate: bool


def concentration_check(iter_count_runs, n_grid, cost_params: CostParams,
                        loop_state: int | None = None) -> ConcentrationReport:
    """Rate at which the per-sample barrier cost C(m, n) = c_rest + c_loop
    mean_{i<n} max_j N_ij settles (analysis.py:281-324; Theorem 1):
    fit log mean_seeds |C(m, n) - C(m, n_max)| against log n.  Runs may be
    device tensors: the prefix means of the row maxima are one cumulative sum
    per run on the device."""
    from scipy import stats
    n_grid = tuple(int(n) for n in n_grid)
    if len(n_grid) < 4:
        raise ValueError("need at least 4 grid points")
    if max(n_grid) / min(n_grid) < 100:
        raise ValueError("grid must span at least two decades")
    costs = cost_params.full_block_costs()
    c_loop = costs[_loop_state(cost_params, loop_state) - 1]
    c_rest = sum(costs) - c_loop
    n_max = max(n_grid)
    if any(run.shape[0] < n_max for run in iter_count_runs):
        raise ValueError("every run must cover the largest grid point")
    idx = np.array(n_grid) - 1
    per_run = []
    for run in iter_count_runs:
        N = _counts(run)
        if isinstance(N, torch.Tensor):
            rowmax = N[:n_max].max(dim=1).values.cpu().numpy()
        else:
            rowmax = N[:n_max].max(axis=1)
        prefix = np.cumsum(rowmax)[idx] / np.array(n_grid, dtype=float)
        per_run.append(c_rest + c_loop * prefix)
    C = np.array(per_run)                                   # [runs, grid]
    limit = float(C[:, -1].mean()) if n_grid[-1] == n_max else float(
        C[:, n_grid.index(n_max)].mean())
    dev = tuple(float(np.mean(np.abs(C[:, g] - limit))) for g in range(len(n_grid)))
    if any(v == 0.0 for v in dev):
        return ConcentrationReport(n_grid, dev, None, None, None, limit, True)
    fit = stats.linregress(np.log(n_grid), np.log(dev))
    half = 1.96 * fit.stderr
    return ConcentrationReport(n_grid=n_grid, deviations=dev, slope=float(fit.slope),
                               slope_stderr=float(fit.stderr),
                               slope_ci95=(float(fit.slope - half), float(fit.slope + half)),
                               limit_estimate=limit, degenerate=False)
