"""Log-density plugins (drop-in for ``fsm_mcmc.targets``).

A :class:`TargetModel` is the plugin boundary (``targets.py:45-60``).  Here
it is a *device descriptor*: a kind from the compiled plugin set plus its
constant tensors in HBM (``fsmc_target`` in ``include/fsmc.h``).  The
constructors compute every constant with the same numpy/scipy calls as the
reference (normalisers, inverse factors, precisions), so the per-evaluation
arithmetic on the device starts from bit-identical inputs.

A per-chain Python callable cannot run on the device (there is no CPU
fallback); a user-defined target is written *batched* instead
(:func:`batched_target`): a torch function of many chains' points at once,
which the engine calls once per round in its batched-evaluation mode.
``log_density`` / ``gradient`` / ``log_density_and_grad`` evaluate through
the device kernel (``fsmc_target_eval``) or that function.
"""

from __future__ import annotations

import ctypes
import math
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

__all__ = [
    "TargetModel", "GaussianPriorDecomposition", "TargetError", "gaussian_target",
    "standard_normal_target", "equicorrelated_covariance", "equicorrelated_gaussian_target",
    "correlated_mog_target", "funnel_target", "gp_classification_data",
    "gp_classification_target", "logistic_residual", "nan_band_target", "flat_target",
    "logistic_regression_data", "logistic_regression_target",
    "conjugate_target", "batched_target",
]

_LOG_2PI = math.log(2.0 * math.pi)


class TargetError(ValueError):
    """Invalid target construction or evaluation input (targets.py:33-34)."""


@dataclass(frozen=True)
class GaussianPriorDecomposition:
    """``p(x) ∝ exp(residual(x)) N(x | 0, chol cholᵀ)`` (targets.py:37-42).

    ``residual_log_density`` is a device TargetModel (the plugin that the
    elliptical kernel evaluates as its shared computation).
    """

    chol: np.ndarray
    residual_log_density: "TargetModel"


@dataclass
class TargetModel:
    """Device log-density plugin (targets.py:45-60)."""

    name: str
    dim: int
    kind: int
    log_norm: float = 0.0
    a: float = 0.0
    b: float = 0.0
    offsets: tuple = ()
    arrays: dict = field(default_factory=dict)      # host float64 arrays
    gaussian_prior: GaussianPriorDecomposition | None = None
    log_density_cost: float = 1.0
    has_gradient: bool = True
    scratch: int = 0               # per-chain shared-memory doubles the plugin needs
    residual_only: bool = False    # evaluates the Gaussian-prior residual, not the density
    _dev: dict = field(default_factory=dict, repr=False)
    _struct: object = field(default=None, repr=False)

    # -- device descriptor ------------------------------------------------
    def device_arrays(self) -> dict:
        dev = torch.cuda.current_device()
        if self._dev.get("_device") != dev:
            self._dev = {"_device": dev}
            for k, v in self.arrays.items():
                self._dev[k] = torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64),
                                               device="cuda")
            if self.gaussian_prior is not None:
                L = np.asarray(self.gaussian_prior.chol, dtype=np.float64)
                self._dev["prior_t"] = torch.as_tensor(np.ascontiguousarray(L.T), device="cuda")
            self._struct = None
        return self._dev

    def struct(self) -> _lib.Target:
        """The ``fsmc_target`` the kernels read (pointers into this model's tensors)."""
        if self._struct is not None and self._dev.get("_device") == torch.cuda.current_device():
            return self._struct
        dev = self.device_arrays()
        t = _lib.Target()
        t.kind = self.kind
        t.dim = self.dim
        t.n_modes = len(self.offsets)
        t.log_norm = self.log_norm
        t.a = self.a
        t.b = self.b
        t.scratch = self.scratch
        for i, o in enumerate(self.offsets):
            t.offsets[i] = o
        for name in ("mean", "diag", "diag2", "mat_t", "mat2_t", "yvec", "data"):
            if name in dev:
                setattr(t, name, dev[name].data_ptr())
        if "data" in self.arrays:
            t.n_rows = int(self.arrays["data"].shape[0])
        t.prior_kind = _lib.PRIOR_NONE
        if self.gaussian_prior is not None:
            L = np.asarray(self.gaussian_prior.chol, dtype=float)
            if np.array_equal(L, np.eye(self.dim)):     # elliptical.py:54
                t.prior_kind = _lib.PRIOR_IDENTITY
            else:
                t.prior_kind = _lib.PRIOR_DENSE
                t.prior_t = dev["prior_t"].data_ptr()
        self._struct = t
        return t

    # -- reference-compatible evaluation ------------------------------------
    def _eval(self, X, grad: bool):
        X = torch.as_tensor(np.asarray(X, dtype=np.float64), device="cuda").reshape(-1, self.dim)
        X = X.contiguous()
        m = X.shape[0]
        lp = torch.empty(m, dtype=torch.float64, device="cuda")
        g = torch.empty_like(X) if grad else None
        if hasattr(self, "batched_evaluator"):     # no per-chain plugin for this design
            self.batched_evaluator(_lib.ESS if self.residual_only else 0)(X, lp, g)
            return lp, g
        t = self.struct()
        fam = _lib.ESS if self.residual_only else 0
        _lib.check(_lib.lib().fsmc_target_eval(ctypes.byref(t), X.data_ptr(), m, lp.data_ptr(),
                                               _lib.ptr(g), fam, 0, _lib.stream_ptr()),
                   "fsmc_target_eval")
        return lp, g

    def log_density(self, x) -> float:
        return _checked(float(self._eval(x, False)[0][0].item()))

    def gradient(self, x) -> np.ndarray:
        return self._eval(x, True)[1][0].cpu().numpy()

    def log_density_and_grad(self, x):
        lp, g = self._eval(x, True)
        return _checked(float(lp[0].item())), g[0].cpu().numpy()

    def log_density_batch(self, X: torch.Tensor, grad: bool = False):
        """Batched device evaluation over rows of X [m, dim]."""
        return self._eval(X, grad)

    def residual(self) -> "TargetModel":
        return self if self.gaussian_prior is None else self.gaussian_prior.residual_log_density


_TARGET_FAILURE_BITS = 0x7ff80000dead0001   # csrc/fsm_device.cuh target_failure()


def _checked(v: float) -> float:
    """Raise TargetError where the plugin could not evaluate (the reference's
    TargetError, e.g. targets.py:213-218) instead of returning its NaN payload."""
    if v != v and struct.unpack("<Q", struct.pack("<d", v))[0] == _TARGET_FAILURE_BITS:
        raise TargetError("kernel matrix not positive definite even with jitter")
    return v


def _check_chol(L, name="covariance factor") -> np.ndarray:
    L = np.asarray(L, dtype=float)
    if L.ndim != 2 or L.shape[0] != L.shape[1]:
        raise TargetError(f"{name} must be square, got shape {L.shape}")
    if np.any(np.triu(L, 1) != 0.0):
        raise TargetError(f"{name} must be lower-triangular")
    if np.any(np.diag(L) <= 0.0):
        raise TargetError(f"{name} needs a positive diagonal")
    return L


def equicorrelated_covariance(d: int, rho: float) -> np.ndarray:
    """targets.py:130-134"""
    if not -1.0 < rho < 1.0:
        raise TargetError(f"correlation must be in (-1, 1), got {rho}")
    return (1.0 - rho) * np.eye(d) + rho * np.ones((d, d))


def _equicorr_params(cov: np.ndarray, rtol: float = 1e-12):
    """(a, b) if cov == a I + b 11^T to rtol, else None."""
    d = cov.shape[0]
    if d < 2:
        return None
    a = float(cov[0, 0] - cov[0, 1])
    b = float(cov[0, 1])
    ref = a * np.eye(d) + b * np.ones((d, d))
    scale = float(np.max(np.abs(cov)))
    if a <= 0 or a + d * b <= 0 or np.max(np.abs(cov - ref)) > rtol * scale:
        return None
    return a, b


def gaussian_target(mean, chol, structure: str = "auto") -> TargetModel:
    """Exact Gaussian N(mean, L Lᵀ) (targets.py:74-122).

    ``structure``: "auto" uses the diagonal plugin for a diagonal factor, the
    O(d) closed form when L Lᵀ = a I + b 11ᵀ, and dense operators otherwise;
    "dense" forces the dense operators (the reference's own arithmetic shape).
    """
    from scipy.linalg import solve_triangular
    mean = np.atleast_1d(np.asarray(mean, dtype=float))
    L = _check_chol(chol)
    d = mean.shape[0]
    if L.shape != (d, d):
        raise TargetError(f"factor shape {L.shape} does not match dim {d}")
    log_norm = -0.5 * d * _LOG_2PI - float(np.sum(np.log(np.diag(L))))
    arrays = {"mean": mean}
    if d == 1:  # targets.py:83-98
        s = float(L[0, 0])
        arrays["diag2"] = np.array([1.0 / (s * s)])
        arrays["diag"] = np.array([1.0 / s])
        return TargetModel(f"gaussian-{d}d", d, _lib.T_GAUSS_DIAG, log_norm, arrays=arrays)
    L_inv = solve_triangular(L, np.eye(d), lower=True)
    prec = L_inv.T @ L_inv
    if structure == "auto" and np.count_nonzero(L - np.diag(np.diag(L))) == 0:
        arrays["diag"] = np.ascontiguousarray(np.diag(L_inv))
        arrays["diag2"] = np.ascontiguousarray(np.diag(prec))
        return TargetModel(f"gaussian-{d}d", d, _lib.T_GAUSS_DIAG, log_norm, arrays=arrays)
    if structure == "auto":
        ab = _equicorr_params(L @ L.T)
        if ab is not None:
            a, b = ab
            return TargetModel(f"gaussian-{d}d", d, _lib.T_GAUSS_EQUICORR, log_norm,
                               a=1.0 / a, b=1.0 / (a + d * b), arrays=arrays)
    arrays["mat_t"] = np.ascontiguousarray(L_inv.T)
    arrays["mat2_t"] = np.ascontiguousarray(prec.T)
    return TargetModel(f"gaussian-{d}d", d, _lib.T_GAUSS_DENSE, log_norm, arrays=arrays)


def standard_normal_target(dim: int = 1) -> TargetModel:
    """targets.py:125-127"""
    return gaussian_target(np.zeros(dim), np.eye(dim))


def equicorrelated_gaussian_target(d: int, rho: float, mean=None) -> TargetModel:
    """N(mean, (1-rho) I + rho 11ᵀ): BASELINE config 3's target, closed form."""
    cov = equicorrelated_covariance(d, rho)
    L = np.linalg.cholesky(cov)
    t = gaussian_target(np.zeros(d) if mean is None else mean, L)
    if t.kind != _lib.T_GAUSS_EQUICORR:  # exact parameters, not re-derived from L L^T
        raise TargetError("equicorrelated detection failed")
    t.a, t.b = 1.0 / (1.0 - rho), 1.0 / (1.0 - rho + d * rho)
    t.name = f"equicorr-gaussian-{d}d-rho{rho}"
    return t


def correlated_mog_target(d: int, rho: float, mode_offsets) -> TargetModel:
    """Equal-weight mixture, modes at o_k 1, shared equicorrelated covariance
    (targets.py:137-188); evaluated in closed form on the device."""
    offsets = np.atleast_1d(np.asarray(mode_offsets, dtype=float))
    if offsets.size < 1:
        raise TargetError("need at least one mode")
    if offsets.size > _lib.MAX_MODES:
        raise TargetError(f"at most {_lib.MAX_MODES} modes are compiled")
    cov = equicorrelated_covariance(d, rho)
    try:
        L = np.linalg.cholesky(cov)
    except np.linalg.LinAlgError as exc:
        raise TargetError(f"singular covariance (d={d}, rho={rho})") from exc
    log_norm = (-0.5 * d * _LOG_2PI - float(np.sum(np.log(np.diag(L)))) - math.log(offsets.size))
    return TargetModel(f"mog-{d}d-rho{rho}", d, _lib.T_MOG, log_norm,
                       a=1.0 / (1.0 - rho), b=1.0 / (1.0 - rho + d * rho),
                       offsets=tuple(float(o) for o in offsets))


def funnel_target(d: int, v_scale: float = 3.0) -> TargetModel:
    """Neal's funnel: v = x[0] ~ N(0, s²), x[i] | v ~ N(0, e^v) (BASELINE config 2).

    Restated for the oracle in tests/golden/make_golden.py (funnel_target)."""
    if d < 2:
        raise TargetError("the funnel needs d >= 2")
    return TargetModel(f"funnel-{d}d", d, _lib.T_FUNNEL, a=float(v_scale))


def nan_band_target(d: int, threshold: float, value: float) -> TargetModel:
    """Fault injection: standard normal that returns ``value`` (NaN / +inf) once x[0] > threshold."""
    return TargetModel(f"nanband-{d}d", d, _lib.T_NANBAND, a=float(threshold), b=float(value))


def box_target(d: int, lo: float = 0.0, hi: float = 1.0) -> TargetModel:
    """Uniform on [lo, hi]^d: log density 0 inside, -inf outside (the compact-support
    target of the reference's slice tests, tests/test_kernels.py:205-212)."""
    if not hi > lo:
        raise TargetError(f"empty box [{lo}, {hi}]")
    return TargetModel(f"box-{d}d", d, _lib.T_BOX, a=float(lo), b=float(hi))


def flat_target(d: int) -> TargetModel:
    return TargetModel(f"flat-{d}d", d, _lib.T_FLAT)


def logistic_residual(y) -> TargetModel:
    """-sum_i log(1 + exp(-y_i x_i)) (numpy ``-logaddexp(0, -y*x).sum()``)."""
    y = np.ascontiguousarray(np.asarray(y, dtype=float))
    return TargetModel(f"logistic-{y.size}", y.size, _lib.T_LOGISTIC, arrays={"yvec": y},
                       has_gradient=True)


def _with_prior(residual: TargetModel, chol, name: str) -> TargetModel:
    L = _check_chol(chol, "prior factor")
    if L.shape != (residual.dim, residual.dim):
        raise TargetError("prior factor does not match the residual dimension")
    return TargetModel(name, residual.dim, residual.kind, residual.log_norm, residual.a,
                       residual.b, residual.offsets, dict(residual.arrays),
                       gaussian_prior=GaussianPriorDecomposition(L, residual),
                       has_gradient=False)


def conjugate_target(dim=2, rho=0.3, lik_mu=0.5, lik_var=0.5) -> TargetModel:
    """Gaussian prior N(0, Σ_rho) times Gaussian likelihood N(x | mu 1, var I): the
    reference's conjugate fixture (pkg/tests/tests_common_conjugate.py:13-29),
    BASELINE config 1's target."""
    prior_cov = equicorrelated_covariance(dim, rho)
    lik = gaussian_target(np.full(dim, lik_mu), np.linalg.cholesky(lik_var * np.eye(dim)))
    return _with_prior(lik, np.linalg.cholesky(prior_cov), "conjugate")


# ------------------------------------------------------- GP hyperparameters
GP_DATA_SEED = 20240617
GP_DATA_THETA = (0.3, 1.0, 1.0)
GP_DEVICE_MAX_ROWS = 56     # per-chain plugin limit (two n x n matrices in shared memory)


def _sq_dists(X: np.ndarray) -> np.ndarray:
    """||x_i - x_j||^2 exactly as targets.py:206-209 forms it (so the device
    reads the reference's own distance matrix)."""
    sq = np.sum(X * X, axis=1)
    d2 = sq[:, None] + sq[None, :] - 2.0 * (X @ X.T)
    np.maximum(d2, 0.0, out=d2)
    return d2


def gp_hyperparameter_target(inputs, outputs, jitter: float = 1e-8,
                             evaluation: str = "auto") -> TargetModel:
    """Posterior over theta = (sigma, tau, lam) of a squared-exponential GP
    regression (targets.py:191-265): K = tau^2 exp(-lam^2 D2) + (sigma^2 +
    jitter) I, N(0, 1) priors, so the Gaussian-prior split has the identity
    factor and the marginal likelihood as residual.  Each evaluation factors
    the chain's own n x n kernel matrix in shared memory (one warp per chain);
    the gradient adds W = L^-1 and the three trace terms.

    ``evaluation``: "plugin" (n <= 56), "batched" (every evaluation and the
    starting points through ``dense.GPHyperEvaluator``: batched fp64
    Cholesky factorizations across chains, any n) or "auto" (the plugin when
    it fits)."""
    X = np.asarray(inputs, dtype=float)
    y = np.ascontiguousarray(np.asarray(outputs, dtype=float))
    if X.ndim != 2 or X.shape[0] < 2:
        raise TargetError("inputs must be an n x p matrix with n >= 2")
    if y.shape != (X.shape[0],):
        raise TargetError(f"outputs shape {y.shape} does not match {X.shape[0]} rows")
    n = X.shape[0]
    if evaluation not in ("auto", "plugin", "batched"):
        raise ValueError("evaluation must be auto, plugin or batched")
    if evaluation == "auto":
        evaluation = "plugin" if n <= GP_DEVICE_MAX_ROWS else "batched"
    if evaluation == "plugin" and n > GP_DEVICE_MAX_ROWS:
        raise TargetError(f"the per-chain GP plugin handles n <= {GP_DEVICE_MAX_ROWS} "
                          f"observations, got {n}")
    arrays = {"data": np.ascontiguousarray(_sq_dists(X)), "yvec": y}
    batched = evaluation == "batched"
    common = dict(name=f"gp-hyper-n{n}", dim=3, kind=_lib.T_GP_HYPER, a=float(jitter),
                  arrays=arrays, scratch=0 if batched else 2 * n * n + 2 * n + 4,
                  log_density_cost=(n / 50.0) ** 3)
    residual = TargetModel(**common, residual_only=True)
    t = TargetModel(**common, gaussian_prior=GaussianPriorDecomposition(np.eye(3), residual))
    if batched:
        from .dense import GPHyperEvaluator

        def batched_evaluator(family=None, _t=t):
            dev = _t.device_arrays()
            return GPHyperEvaluator(dev["data"], dev["yvec"], jitter,
                                    residual=family == _lib.ESS)
        t.batched_evaluator = batched_evaluator
        residual.batched_evaluator = lambda family=None, _t=t: batched_evaluator(_lib.ESS)
    return t


def make_synthetic_gp_dataset(n: int = 50, p: int = 3, seed: int = GP_DATA_SEED,
                              theta=GP_DATA_THETA):
    """(inputs, outputs) drawn from the GP model at fixed hyperparameters
    (targets.py:273-287; same numpy draws, so the same data)."""
    if n < 2:
        raise TargetError("need n >= 2 data points")
    sigma, tau, lam = theta
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n, p))
    Kf = (tau * tau) * np.exp(-(lam * lam) * _sq_dists(X)) + 1e-10 * np.eye(n)
    f = np.linalg.cholesky(Kf) @ rng.normal(size=n)
    return X, f + sigma * rng.normal(size=n)


def save_gp_dataset_csv(path, X, y) -> None:
    """Feature columns then the output, one header line (targets.py:290-294)."""
    X = np.asarray(X, dtype=float)
    header = ",".join([f"x{i}" for i in range(X.shape[1])] + ["y"])
    np.savetxt(path, np.column_stack([X, y]), delimiter=",", header=header, comments="")


def load_gp_dataset_csv(path):
    data = np.loadtxt(path, delimiter=",", skiprows=1)
    return data[:, :-1], data[:, -1]


def logistic_regression_data(n_obs: int = 100_000, d: int = 256, seed: int = 0):
    """Synthetic Bayesian logistic regression (BASELINE config 5; SURVEY.md
    Appendix B): X ~ N(0,1)/sqrt(d), theta* ~ N(0, I), y ~ Bernoulli(sigmoid(X theta*))."""
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n_obs, d)) / math.sqrt(d)
    theta = rng.normal(size=d)
    y = (rng.uniform(size=n_obs) < 1.0 / (1.0 + np.exp(-(X @ theta)))).astype(float)
    return X, y


def logistic_regression_target(X, y) -> TargetModel:
    """log p(theta) = sum_i [y_i z_i - log(1 + e^{z_i})] - theta.theta/2 with
    z = X theta; gradient X^T (y - sigmoid(z)) - theta.  Restated for the
    oracle in tests/golden/make_golden.py (logreg_target)."""
    X = np.ascontiguousarray(np.asarray(X, dtype=float))
    y = np.ascontiguousarray(np.asarray(y, dtype=float))
    if X.ndim != 2 or y.shape != (X.shape[0],):
        raise TargetError("need X [n, d] and y [n]")
    return TargetModel(f"logreg-{X.shape[0]}x{X.shape[1]}", X.shape[1], _lib.T_LOGREG,
                       arrays={"data": X, "yvec": y})


def gp_classification_data(n_pts: int, seed: int = 20240617):
    """Synthetic GP-classification latent problem:
    RBF kernel on N(0, I_2) inputs, latent f = L eps, labels ±1 by sigma(f)."""
    rng = np.random.default_rng(seed)
    S = rng.normal(size=(n_pts, 2))
    sq = np.sum(S * S, axis=1)
    d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * (S @ S.T), 0.0)
    K = np.exp(-0.5 * d2) + 1e-6 * np.eye(n_pts)
    L = np.linalg.cholesky(K)
    f = L @ rng.normal(size=n_pts)
    y = np.where(rng.uniform(size=n_pts) < 1.0 / (1.0 + np.exp(-f)), 1.0, -1.0)
    return L, y


def gp_classification_target(n_pts: int = 1024, seed: int = 20240617) -> TargetModel:
    """BASELINE config 4's latent target in f-space: prior N(0, K = L Lᵀ),
    residual -sum log(1 + exp(-y f))."""
    L, y = gp_classification_data(n_pts, seed)
    return _with_prior(logistic_residual(y), L, f"gpc-{n_pts}")


def batched_target(name: str, dim: int, log_density=None, log_density_and_grad=None,
                   gaussian_prior=None, log_density_cost: float = 1.0) -> TargetModel:
    """A user-defined target, the plugin ``TargetModel(name, dim, log_density,
    gradient, log_density_and_grad, gaussian_prior)`` (targets.py:45-60) in
    batched form: every callable takes the points of many chains at once as a
    float64 CUDA tensor ``theta [k, dim]`` and returns torch tensors --
    ``log_density(theta) -> lp [k]``, ``log_density_and_grad(theta) -> (lp [k],
    grad [k, dim])`` (needed by NUTS).  ``gaussian_prior=(chol, residual)``
    (the elliptical kernel's split, targets.py:37-42) takes the prior factor
    and the batched residual log density.

    The engine runs such a target in its batched-evaluation mode: chains
    advance on the device to their next log-density request, the requests of
    a round are evaluated in one call of these functions, the chains resume;
    starting points likewise (deferred init).  NaN / +inf results raise the
    reference's BlockFailure as for the device plugins."""
    if log_density is None and log_density_and_grad is None:
        raise TargetError("batched_target needs log_density or log_density_and_grad")
    dim = int(dim)

    def full(theta, lp, g):
        if g is not None:
            if log_density_and_grad is None:
                raise TargetError(f"target {name!r} has no gradient (log_density_and_grad)")
            v, gr = log_density_and_grad(theta)
            g.copy_(gr)
        else:
            v = log_density(theta) if log_density is not None else log_density_and_grad(theta)[0]
        lp.copy_(v)

    prior = None
    residual = None
    if gaussian_prior is not None:
        chol, res_fn = gaussian_prior
        residual = TargetModel(f"{name}-residual", dim, _lib.T_EXTERNAL, residual_only=True,
                               has_gradient=False, log_density_cost=log_density_cost)

        def res(theta, lp, g):
            lp.copy_(res_fn(theta))
        residual.batched_evaluator = lambda family=None: res
        prior = GaussianPriorDecomposition(_check_chol(chol, "prior factor"), residual)
    t = TargetModel(name, dim, _lib.T_EXTERNAL, gaussian_prior=prior,
                    has_gradient=log_density_and_grad is not None,
                    log_density_cost=log_density_cost)

    def batched_evaluator(family=None):
        if family == _lib.ESS and residual is not None:
            return residual.batched_evaluator()
        return full
    t.batched_evaluator = batched_evaluator
    return t
