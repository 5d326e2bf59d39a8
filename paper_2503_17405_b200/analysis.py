"""Cross-chain diagnostics on the device (drop-in for ``fsm_mcmc.analysis``'s ESS).

``effective_sample_size`` follows ``analysis.py:336-418``: per-chain
autocovariances, a chain-mean based var+, Geyer's initial positive pairs with
the monotone fix, ESS = min(m n / tau, m n), pooled = min over dimensions.
The partial sums (per-chain means, summed lag-t autocovariances) come from
``fsmc_diag_partials`` in tiles of 32 lags, fetched only as far as Geyer's
truncation needs.  The same partials are what the multi-GPU path all-reduces
(``distributed.py``), so 1 GPU is the world-size-1 case of one code path.

``rhat`` is Gelman-Rubin's potential scale reduction sqrt(var+ / W) from the
same moments (new: the reference has none).
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _lib

__all__ = ["EssSummary", "effective_sample_size", "rhat", "DiagMoments", "diag_moments",
           "ess_from_moments", "rhat_from_moments", "LAG_TILE"]

LAG_TILE = 32


@dataclass(frozen=True)
class EssSummary:
    per_dimension: tuple
    pooled: float           # min across dimensions
    per_cost: float | None
    per_second: float | None
    flagged: bool           # capped/floored somewhere


@dataclass
class DiagMoments:
    """Everything ESS / R-hat need, summed over the chains it covers.

    n: rows per chain; m: chains; sum_mean [d]; var_means [d] (ddof=1 across
    chains); max_chain_var [d]; acov_tile(k) -> [32, d] sums over chains of the
    lag 32k..32k+31 autocovariances (each / n, analysis.py:344-347).
    """

    n: int
    m: int
    d: int
    var_means: np.ndarray
    max_chain_var: np.ndarray
    acov_tile: Callable[[int], np.ndarray]
    acov_all: Callable[[], np.ndarray] | None = None   # [n, d] sums over chains, all lags


def _as_device(chains) -> torch.Tensor:
    if isinstance(chains, torch.Tensor):
        t = chains.to(device="cuda", dtype=torch.float64)
    else:
        t = torch.as_tensor(np.asarray(chains, dtype=np.float64), device="cuda")
    if t.dim() == 2:
        t = t[:, :, None]
    if t.dim() != 3:
        raise ValueError(f"expected an (n, m, d) array, got shape {tuple(t.shape)}")
    return t.contiguous()


def diag_moments(chains, burn: int = 0) -> DiagMoments:
    """Per-device partial moments of samples [n, m, d] (rows burn..n-1)."""
    S = _as_device(chains)
    n_all, m, d = S.shape
    n = n_all - burn
    lib = _lib.lib()
    mean = torch.empty((m, d), dtype=torch.float64, device="cuda")
    var = torch.empty((m, d), dtype=torch.float64, device="cuda")
    tile = torch.empty((LAG_TILE, d), dtype=torch.float64, device="cuda")
    _lib.check(lib.fsmc_diag_partials(S.data_ptr(), n_all, m, d, burn, 0, LAG_TILE,
                                      mean.data_ptr(), tile.data_ptr(), var.data_ptr(),
                                      _lib.stream_ptr()), "fsmc_diag_partials")
    first = tile.cpu().numpy()
    var_means = mean.var(dim=0, unbiased=True).cpu().numpy() if m > 1 else np.zeros(d)
    chain_var = var.amax(dim=0).cpu().numpy()

    def acov_tile(k: int) -> np.ndarray:
        if k == 0:
            return first
        _lib.check(lib.fsmc_diag_partials(S.data_ptr(), n_all, m, d, burn, k * LAG_TILE,
                                          LAG_TILE, mean.data_ptr(), tile.data_ptr(), None,
                                          _lib.stream_ptr()), "fsmc_diag_partials")
        return tile.cpu().numpy()

    def acov_all() -> np.ndarray:
        """Every lag at once by FFT (analysis.py:344-347), for slowly mixing
        chains whose Geyer truncation needs many lag tiles."""
        # sum_j acov_j = irfft(sum_j |F_j|^2): the power spectra are summed over
        # chains first, so one inverse transform per dimension remains
        # (transforms along the contiguous last axis: 1.5x faster than along dim 0)
        size = 1 << int(math.ceil(math.log2(2 * n)))
        power = torch.zeros((d, size // 2 + 1), dtype=torch.float64, device="cuda")
        chunk = max(1, (1 << 27) // (size * d))   # ~2 GB of complex work at a time
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            c = (S[burn:, lo:hi, :] - mean[lo:hi]).permute(1, 2, 0)   # [chains, d, n]
            f = torch.fft.rfft(c, n=size, dim=2)
            r = torch.view_as_real(f)                  # one product and one reduction
            power += (r * r).sum(dim=(0, 3))           # pass (tools/acov_probe.py: -11%)
        return (torch.fft.irfft(power, n=size, dim=1)[:, :n] / n).T.cpu().numpy()

    return DiagMoments(n=n, m=m, d=d, var_means=var_means, max_chain_var=chain_var,
                       acov_tile=acov_tile, acov_all=acov_all)


class _Acov:
    """Mean (over chains) autocovariance of one dimension set: lag tiles on
    demand, switching to one FFT over every lag once the truncation point is
    beyond a few tiles and the tiles left to reach n cost more than the FFT."""

    TILE_LIMIT = 3
    # one all-lags transform costs about as much as this many lag-tile passes
    # (tools/acov_probe.py: 45 ms against 1.7 ms per tile at C3's size), so
    # short chains (C4: n = 180 rows, 6 tiles in all) stay on the tiles
    FFT_TILE_EQUIV = 16

    def __init__(self, mom: DiagMoments):
        self.mom = mom
        self.tiles: list[np.ndarray] = []
        self.full = None

    def __call__(self, t: int, k: int) -> float:
        if self.full is not None:
            return float(self.full[t, k]) if t < self.full.shape[0] else 0.0
        tile = t // LAG_TILE
        if (tile >= self.TILE_LIMIT and self.mom.acov_all is not None
                and -(-self.mom.n // LAG_TILE) - len(self.tiles) > self.FFT_TILE_EQUIV):
            self.full = self.mom.acov_all() / self.mom.m
            return self(t, k)
        while len(self.tiles) <= tile:
            self.tiles.append(self.mom.acov_tile(len(self.tiles)) / self.mom.m)
        return float(self.tiles[tile][t % LAG_TILE, k])


def _ess_dim(ac: _Acov, mom: DiagMoments, k: int) -> tuple[float, bool]:
    """analysis.py:336-386 for dimension k."""
    m, n = mom.m, mom.n
    total = m * n
    if mom.max_chain_var[k] <= 1e-8:   # np.allclose(var, 0)
        warnings.warn("constant chain: ESS floored to 1", stacklevel=3)
        return 1.0, True
    mean_var = ac(0, k) * n / (n - 1.0)
    var_plus = mean_var * (n - 1.0) / n
    if m > 1:
        var_plus += float(mom.var_means[k])
    rho = {0: 1.0}
    rho_even = 1.0
    rho_odd = 1.0 - (mean_var - ac(1, k)) / var_plus
    rho[1] = rho_odd
    anticorrelated = (rho_even + rho_odd) < 0.0
    t = 1
    while t < n - 2 and (rho_even + rho_odd) >= 0.0:
        rho_even = 1.0 - (mean_var - ac(t + 1, k)) / var_plus
        rho_odd = 1.0 - (mean_var - ac(t + 2, k)) / var_plus
        rho[t + 1] = rho_even
        if (rho_even + rho_odd) >= 0.0:
            rho[t + 2] = rho_odd
        t += 2
    max_t = t
    t = 1
    while t <= max_t - 2:   # initial monotone sequence
        if rho.get(t + 1, 0.0) + rho.get(t + 2, 0.0) > rho.get(t - 1, 0.0) + rho.get(t, 0.0):
            rho[t + 1] = (rho.get(t - 1, 0.0) + rho.get(t, 0.0)) / 2.0
            rho[t + 2] = rho[t + 1]
        t += 2
    # numpy's pairwise sum over the zero-filled rho[:max_t] (analysis.py:378)
    tau = -1.0 + 2.0 * float(np.array([rho.get(i, 0.0) for i in range(max_t)]).sum()) + \
        (rho.get(max_t + 1, 0.0) if max_t + 1 < n else 0.0)
    flagged = False
    if tau <= 0 or not math.isfinite(tau):
        tau = 1.0 / total
        flagged = True
    ess = total / tau
    if anticorrelated:
        warnings.warn("anticorrelated chain: ESS capped at the sample count", stacklevel=3)
        flagged = True
    return float(min(ess, float(total))), flagged


def _geyer_all(acf: np.ndarray, mom: DiagMoments) -> tuple[np.ndarray, np.ndarray]:
    """`_ess_dim` for every dimension at once (numpy over dimensions, the
    same floating-point operations in the same order).  acf [T, d]: mean
    autocovariances for lags 0..T-1, T large enough that every dimension's
    initial positive sequence ends inside it or T == n.  Returns (ess [d],
    flagged [d]); constant chains are handled by the caller."""
    m, n = mom.m, mom.n
    total = float(m * n)
    T, d = acf.shape
    mean_var = acf[0] * n / (n - 1.0)
    var_plus = mean_var * (n - 1.0) / n
    if m > 1:
        var_plus = var_plus + mom.var_means
    rho = 1.0 - (mean_var[None, :] - acf) / var_plus[None, :]
    rho[0] = 1.0
    npairs = (T + 1) // 2
    if 2 * npairs > T:
        rho = np.vstack([rho, np.zeros((1, d))])
    P = rho[0::2][:npairs] + rho[1::2][:npairs]          # pair sums, pair j = (2j, 2j+1)
    anticorrelated = P[0] < 0.0
    # pairs computed by the reference loop: j = 1 .. J, J = first j >= 1 with
    # P_j < 0, or the last j with 2j - 1 < n - 2
    j_lim = max(0, (n - 2) // 2)                       # largest j with 2j - 1 < n - 2
    js = np.arange(npairs)[:, None]
    # the reference loop runs while a pair sum is >= 0: a NaN pair stops it too
    neg = ~(P >= 0.0) & (js >= 1) & (js <= j_lim)
    first_neg = np.where(neg.any(axis=0), neg.argmax(axis=0), j_lim)
    J = np.where(~(P[0] >= 0.0), 0, first_neg)                     # [d]
    odd_kept = (js < J[None, :]) | ((js == J[None, :]) & (P >= 0.0))  # rho[2j+1] stored?
    Pm = rho[0::2][:npairs] + np.where(odd_kept | (js == 0), rho[1::2][:npairs], 0.0)
    # initial monotone sequence over pairs 1..J: running minimum of pair sums
    # (pair j takes the minimum so far when it exceeds it: a cumulative minimum;
    # min is exact, so the values equal the reference loop's)
    cm = np.minimum.accumulate(Pm, axis=0)
    act = (js >= 1) & (js <= J[None, :])
    modified = np.zeros_like(Pm, dtype=bool)
    modified[1:] = act[1:] & (Pm[1:] > cm[:-1])
    run = np.where(act, cm, Pm)
    ev = np.where(modified, run / 2.0, rho[0::2][:npairs])
    od = np.where(modified, run / 2.0, np.where(odd_kept | (js == 0), rho[1::2][:npairs], 0.0))
    # tau = -1 + 2 sum_{i < 2J+1} rho_i: numpy's pairwise sum of each
    # dimension's contiguous rho[:max_t] (analysis.py:378)
    seq = np.empty((d, 2 * npairs))
    seq[:, 0::2], seq[:, 1::2] = ev.T, od.T
    # dimensions with the same length sum together: a reduction along the
    # contiguous last axis runs the same pairwise sum per row
    lengths = np.unique(J)
    if 4 * lengths.size <= d:
        S = np.empty(d)
        for L in lengths:
            ks = np.nonzero(J == L)[0]
            S[ks] = np.ascontiguousarray(seq[ks, :2 * L + 1]).sum(axis=1)
    else:
        S = np.array([seq[k, :2 * J[k] + 1].sum() for k in range(d)])
    tau = -1.0 + 2.0 * S
    bad = (tau <= 0) | ~np.isfinite(tau)
    tau = np.where(bad, 1.0 / total, tau)
    ess = np.minimum(total / tau, total)
    return ess, bad, anticorrelated


def _acf_for_geyer(mom: DiagMoments) -> np.ndarray:
    """Mean autocovariances [T, d] far enough for every dimension's initial
    positive sequence: lag tiles until each dimension's pair sums turn
    negative, one FFT over every lag beyond a few tiles."""
    n = mom.n
    tiles = []
    with np.errstate(divide="ignore", invalid="ignore"):
        acf = _acf_tiles(mom, tiles)
    if acf is not None:
        return acf
    if _fft_pays(mom, len(tiles)):
        return mom.acov_all()[:n] / mom.m
    while len(tiles) * LAG_TILE < n:
        tiles.append(mom.acov_tile(len(tiles)) / mom.m)
    return np.vstack(tiles)[:n]


def _fft_pays(mom: DiagMoments, tiles_done: int) -> bool:
    """The all-lags transform beats the lag tiles still needed to reach n."""
    return (mom.acov_all is not None
            and -(-mom.n // LAG_TILE) - tiles_done > _Acov.FFT_TILE_EQUIV)


def _acf_tiles(mom: DiagMoments, tiles: list):
    n = mom.n
    for k in range(_Acov.TILE_LIMIT):
        tiles.append(mom.acov_tile(k) / mom.m)
        acf = np.vstack(tiles)[:n]
        if acf.shape[0] >= n:
            return acf
        mean_var = acf[0] * n / (n - 1.0)
        var_plus = mean_var * (n - 1.0) / n + (mom.var_means if mom.m > 1 else 0.0)
        rho = 1.0 - (mean_var[None, :] - acf) / var_plus[None, :]
        rho[0] = 1.0
        h = acf.shape[0] // 2
        P = rho[0:2 * h:2] + rho[1:2 * h:2]
        done = ((P < 0.0) | ~np.isfinite(P)).any(axis=0)
        if bool(done.all()):
            return acf
        # a dimension still correlated at 0.5 at the last lag fetched will need
        # far more tiles: go to the all-lags transform at once
        if _fft_pays(mom, len(tiles)) and bool((rho[-1][~done] > 0.5).any()):
            return None
    return None


def ess_from_moments(mom: DiagMoments, model_cost=None, walltime=None) -> EssSummary:
    const = np.asarray(mom.max_chain_var) <= 1e-8        # np.allclose(var, 0)
    if const.any():
        warnings.warn("constant chain: ESS floored to 1", stacklevel=2)
    with np.errstate(divide="ignore", invalid="ignore"):
        ess, bad, anti = _geyer_all(_acf_for_geyer(mom), mom)
    if (anti & ~const).any():
        warnings.warn("anticorrelated chain: ESS capped at the sample count", stacklevel=2)
    ess = np.where(const, 1.0, ess)
    per_dim = [float(v) for v in ess]
    flagged = bool(const.any() or (bad | anti)[~const].any())
    pooled = min(per_dim)
    return EssSummary(per_dimension=tuple(per_dim), pooled=pooled,
                      per_cost=pooled / model_cost if model_cost else None,
                      per_second=pooled / walltime if walltime else None, flagged=flagged)


def effective_sample_size(chains, model_cost: float | None = None,
                          walltime: float | None = None, burn: int = 0) -> EssSummary:
    """Autocorrelation-adjusted sample count of an (n, m, d) array (analysis.py:389-418)."""
    shape = tuple(chains.shape)
    n = shape[0] - burn
    if len(shape) not in (2, 3):
        raise ValueError(f"expected an (n, m, d) array, got shape {shape}")
    if n < 10:
        raise ValueError(f"need at least 10 samples per chain, got {n}")
    return ess_from_moments(diag_moments(chains, burn), model_cost, walltime)


def rhat_from_moments(mom: DiagMoments) -> np.ndarray:
    """Potential scale reduction sqrt(var+ / W) per dimension."""
    tile0 = mom.acov_tile(0)[0] / mom.m
    n = mom.n
    W = tile0 * n / (n - 1.0)
    var_plus = W * (n - 1.0) / n + (mom.var_means if mom.m > 1 else 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.sqrt(var_plus / W)


def rhat(chains, burn: int = 0) -> np.ndarray:
    """Gelman-Rubin R-hat per dimension of an (n, m, d) array."""
    return rhat_from_moments(diag_moments(chains, burn))


# the cost-theory half of the reference module (analysis.py:53-324)
from .efficiency import (BoundEstimate, ConcentrationReport, EfficiencyReport,  # noqa: E402
                         PropBoundReport, barrier_cost, bernoulli_bound_closed_form, bound_R,
                         concentration_check, desync_cost, efficiency_model, efficiency_report,
                         hoeffding_rate, verify_prop_bound)

__all__ += ["barrier_cost", "desync_cost", "efficiency_model", "efficiency_report",
            "EfficiencyReport", "bound_R", "BoundEstimate", "bernoulli_bound_closed_form",
            "verify_prop_bound", "PropBoundReport", "concentration_check", "ConcentrationReport",
            "hoeffding_rate"]
