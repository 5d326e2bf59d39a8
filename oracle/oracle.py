"""ctypes wrapper around ``oracle/liboracle.so`` -- TEST INFRASTRUCTURE ONLY.

The oracle is the CPU restatement of the reference's sampling path
(``oracle/fsm_oracle.c``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (``cpu_baseline`` leg, ``--impl reference``) may import this
module, and only as the checker / CPU baseline.  Parity of the oracle itself
is pinned by ``tests/test_oracle_golden.py`` against fixtures frozen from the
live reference (``tests/golden/make_golden.py``).

Target constructors compute their constants with the same numpy/scipy calls
the reference uses (``targets.py:74-188``), so the C side only restates the
per-evaluation arithmetic.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
LOG_2PI = math.log(2.0 * math.pi)

DRMH, ESS, NUTS, SLICE = 1, 2, 3, 4
VARIANTS = {"plain": 0, "bundled": 1, "amortized": 2}
T_GAUSS, T_MOG, T_FUNNEL, T_NANBAND, T_LOGISTIC, T_FLAT, T_LOGREG, T_BOX, T_GP = range(1, 10)


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "fsm_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-C", HERE, "-s"])
    return LIB_PATH


_P = ctypes.POINTER(ctypes.c_double)
_PI64 = ctypes.POINTER(ctypes.c_int64)


class _Target(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("dim", ctypes.c_int32), ("n_modes", ctypes.c_int32),
                ("residual", ctypes.c_int32), ("log_norm", ctypes.c_double),
                ("p0", ctypes.c_double), ("p1", ctypes.c_double),
                ("mean", _P), ("L_inv", _P), ("prec", _P), ("modes", _P), ("yvec", _P),
                ("prior_chol", _P), ("prior_identity", ctypes.c_int32), ("pad1", ctypes.c_int32),
                ("data", _P), ("n_rows", ctypes.c_int64)]


class _Kernel(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("max_tries", ctypes.c_int32),
                ("proposal_scale", ctypes.c_double), ("step_size", ctypes.c_double),
                ("max_depth", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("divergence_threshold", ctypes.c_double), ("slice_width", ctypes.c_double),
                ("max_expansions", ctypes.c_int32), ("pad2", ctypes.c_int32)]


class _Error(ctypes.Structure):
    _fields_ = [("chain", ctypes.c_int64), ("iteration", ctypes.c_int64), ("tick", ctypes.c_int64),
                ("kind", ctypes.c_int32), ("label", ctypes.c_int32)]


class _Out(ctypes.Structure):
    _fields_ = [("samples", _P), ("loop_counts", _PI64), ("sample_ticks", _PI64),
                ("block_counts", _PI64), ("tick_count", ctypes.c_int64),
                ("native_shared", ctypes.c_int64), ("budget_exceeded", ctypes.c_int64),
                ("n_done", ctypes.c_int64), ("sample_counts", _PI64), ("err", _Error)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.or_bits.restype = ctypes.c_uint64
        _lib.or_bits.argtypes = [ctypes.c_uint64] * 3
        _lib.or_mix64.restype = ctypes.c_uint64
        _lib.or_mix64.argtypes = [ctypes.c_uint64]
        _lib.or_split_stream.restype = ctypes.c_uint64
        _lib.or_split_stream.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        for f in ("or_uniform", "or_normal"):
            getattr(_lib, f).restype = ctypes.c_double
            getattr(_lib, f).argtypes = [ctypes.c_uint64] * 3
        _lib.or_ndtri.restype = ctypes.c_double
        _lib.or_ndtri.argtypes = [ctypes.c_double]
        _lib.or_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
        _lib.or_log_density.restype = ctypes.c_double
        _lib.or_log_density_grad.restype = ctypes.c_double
        _lib.or_run_fsm.argtypes = [ctypes.POINTER(_Kernel), ctypes.POINTER(_Target),
                                    ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, _P,
                                    ctypes.c_double, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_int32), ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                    ctypes.POINTER(_Out)]
        _lib.or_run_standard.argtypes = [ctypes.POINTER(_Kernel), ctypes.POINTER(_Target),
                                         ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, _P,
                                         ctypes.c_double, ctypes.c_int64, ctypes.c_int32,
                                         ctypes.POINTER(_Out)]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


# ------------------------------------------------------------------ targets
@dataclass
class OracleTarget:
    kind: int
    dim: int
    n_modes: int = 0
    log_norm: float = 0.0
    p0: float = 0.0
    p1: float = 0.0
    arrays: dict = field(default_factory=dict)
    prior_identity: bool = False
    residual: bool = False     # GP: evaluate the marginal likelihood only

    def struct(self) -> _Target:
        a = self.arrays
        t = _Target(kind=self.kind, dim=self.dim, n_modes=self.n_modes, log_norm=self.log_norm,
                    p0=self.p0, p1=self.p1, prior_identity=int(self.prior_identity),
                    residual=int(self.residual))
        for name in ("mean", "L_inv", "prec", "modes", "yvec", "prior_chol", "data"):
            if a.get(name) is not None:
                setattr(t, name, _ptr(a[name]))
        if a.get("data") is not None:
            t.n_rows = a["data"].shape[0]
        return t

    def log_density(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        ts = self.struct()
        lib().or_log_density.argtypes = [ctypes.POINTER(_Target), _P]
        return lib().or_log_density(ctypes.byref(ts), _ptr(x))

    def log_density_and_grad(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.empty(self.dim)
        ts = self.struct()
        lib().or_log_density_grad.argtypes = [ctypes.POINTER(_Target), _P, _P]
        lp = lib().or_log_density_grad(ctypes.byref(ts), _ptr(x), _ptr(g))
        return lp, g


def gaussian(mean, chol) -> OracleTarget:
    """targets.py:74-122"""
    from scipy.linalg import solve_triangular
    mean = np.atleast_1d(np.asarray(mean, dtype=float))
    L = np.asarray(chol, dtype=float)
    d = mean.shape[0]
    log_norm = -0.5 * d * LOG_2PI - float(np.sum(np.log(np.diag(L))))
    if d == 1:
        s = float(L[0, 0])
        prec = np.array([[1.0 / (s * s)]])
        L_inv = np.array([[1.0 / s]])
    else:
        L_inv = solve_triangular(L, np.eye(d), lower=True)
        prec = L_inv.T @ L_inv
    return OracleTarget(T_GAUSS, d, log_norm=log_norm,
                        arrays={"mean": np.ascontiguousarray(mean), "L_inv": np.ascontiguousarray(L_inv),
                                "prec": np.ascontiguousarray(prec)})


def equicorrelated_covariance(d, rho):
    """targets.py:130-134"""
    return (1.0 - rho) * np.eye(d) + rho * np.ones((d, d))


def mog(d, rho, offsets) -> OracleTarget:
    """targets.py:137-188"""
    from scipy.linalg import cho_solve
    offsets = np.atleast_1d(np.asarray(offsets, dtype=float))
    cov = equicorrelated_covariance(d, rho)
    L = np.linalg.cholesky(cov)
    prec = cho_solve((L, True), np.eye(d))
    modes = offsets[:, None] * np.ones(d)[None, :]
    log_norm = (-0.5 * d * LOG_2PI - float(np.sum(np.log(np.diag(L)))) - math.log(offsets.size))
    return OracleTarget(T_MOG, d, n_modes=offsets.size, log_norm=log_norm,
                        arrays={"prec": np.ascontiguousarray(prec),
                                "modes": np.ascontiguousarray(modes)})


def funnel(d, v_scale=3.0) -> OracleTarget:
    return OracleTarget(T_FUNNEL, d, p0=float(v_scale))


def nanband(d, threshold, value) -> OracleTarget:
    return OracleTarget(T_NANBAND, d, p0=float(threshold), p1=float(value))


def flat(d) -> OracleTarget:
    return OracleTarget(T_FLAT, d)


def box(d, lo=0.0, hi=1.0) -> OracleTarget:
    """0 on [lo, hi]^d, -inf outside (pkg/tests/test_kernels.py:205-212)."""
    return OracleTarget(T_BOX, d, p0=float(lo), p1=float(hi))


def logreg(X, y) -> OracleTarget:
    """Bayesian logistic regression, N(0, I) prior (tests/golden/make_golden.py logreg_target)."""
    X = np.ascontiguousarray(np.asarray(X, dtype=float))
    y = np.ascontiguousarray(np.asarray(y, dtype=float))
    return OracleTarget(T_LOGREG, X.shape[1], arrays={"data": X, "yvec": y})


def gp_hyper(X, y, jitter=1e-8) -> OracleTarget:
    """GP hyperparameter posterior (targets.py:191-265); the squared distances are
    formed exactly as the reference forms them, so C starts from the same matrix.
    The elliptical kernel evaluates its marginal likelihood (identity prior)."""
    X = np.asarray(X, dtype=float)
    sq = np.sum(X * X, axis=1)
    d2 = sq[:, None] + sq[None, :] - 2.0 * (X @ X.T)
    np.maximum(d2, 0.0, out=d2)
    t = OracleTarget(T_GP, 3, p0=float(jitter),
                     arrays={"data": np.ascontiguousarray(d2),
                             "yvec": np.ascontiguousarray(np.asarray(y, dtype=float))})
    t.arrays["prior_chol"] = np.eye(3)
    t.prior_identity = True
    return t


def with_prior(residual: OracleTarget, chol) -> OracleTarget:
    """Gaussian-prior split (targets.py:37-42) for the elliptical kernel."""
    L = np.ascontiguousarray(np.asarray(chol, dtype=float))
    residual.arrays["prior_chol"] = L
    residual.prior_identity = bool(np.array_equal(L, np.eye(L.shape[0])))
    return residual


def conjugate(dim=2, rho=0.3, lik_mu=0.5, lik_var=0.5) -> OracleTarget:
    """pkg/tests/tests_common_conjugate.py:13-29"""
    prior_cov = equicorrelated_covariance(dim, rho)
    lik = gaussian(np.full(dim, lik_mu), np.linalg.cholesky(lik_var * np.eye(dim)))
    return with_prior(lik, np.linalg.cholesky(prior_cov))


def logistic_fspace(L, y) -> OracleTarget:
    """GP-classification latent, f-space form: prior N(0, L L^T), residual
    -sum logaddexp(0, -y * f)."""
    y = np.ascontiguousarray(np.asarray(y, dtype=float))
    return with_prior(OracleTarget(T_LOGISTIC, y.shape[0], arrays={"yvec": y}), L)


# ------------------------------------------------------------------ kernels
def drmh(max_tries, proposal_scale):
    return _Kernel(family=DRMH, max_tries=int(max_tries), proposal_scale=float(proposal_scale))


def elliptical():
    return _Kernel(family=ESS)


def nuts(step_size, max_depth=10, divergence_threshold=1000.0):
    return _Kernel(family=NUTS, step_size=float(step_size), max_depth=int(max_depth),
                   divergence_threshold=float(divergence_threshold))


def slice_(initial_width, max_expansions=32):
    """kernels/slice_sampling.py:50"""
    return _Kernel(family=SLICE, slice_width=float(initial_width),
                   max_expansions=int(max_expansions))


def loop_states(kernel):
    if kernel.family == SLICE:
        return (2, 4)
    return (2, 3, 4) if kernel.family == NUTS else (2,)


class OracleError(RuntimeError):
    def __init__(self, err):
        super().__init__(f"chain {err.chain}, sample index {err.iteration}: kind {err.kind} "
                         f"label {err.label}")
        self.chain, self.iteration, self.tick = err.chain, err.iteration, err.tick
        self.kind, self.label = err.kind, err.label


class OracleBudget(RuntimeError):
    def __init__(self, result):
        super().__init__("tick budget exceeded")
        self.result = result


def _run(fn, kernel, target, m, n, seed, x0, init_jitter, chain_offset, nthreads, extra):
    d = target.dim
    K = 5 if kernel.family in (NUTS, SLICE) else 3
    L = len(loop_states(kernel))
    samples = np.zeros((n, m, d))
    loops = np.zeros((L, n, m), dtype=np.int64)
    ticks = np.zeros((n, m), dtype=np.int64)
    blocks = np.zeros(K, dtype=np.int64)
    counts = np.zeros(m, dtype=np.int64)
    out = _Out(samples=_ptr(samples), loop_counts=loops.ctypes.data_as(_PI64),
               sample_ticks=ticks.ctypes.data_as(_PI64), block_counts=blocks.ctypes.data_as(_PI64),
               sample_counts=counts.ctypes.data_as(_PI64))
    ts = target.struct()
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    rc = fn(ctypes.byref(kernel), ctypes.byref(ts), m, seed & (2**64 - 1), chain_offset,
            _ptr(x0a), float(init_jitter), n, *extra, nthreads, ctypes.byref(out))
    iters = loops[1] if kernel.family == NUTS else (loops[0] + loops[1] if kernel.family == SLICE
                                                    else loops[0])
    res = {"samples": samples, "iter_counts": iters,
           "loop_counts": {s: loops[i] for i, s in enumerate(loop_states(kernel))},
           "sample_ticks": ticks, "block_exec_counts": blocks, "tick_count": out.tick_count,
           "native_shared_evals": out.native_shared, "sample_counts": counts,
           "n_done": out.n_done}
    if rc == 1:
        raise OracleError(out.err)
    if rc == 2:
        nd = out.n_done
        res["samples"] = samples[:nd]
        res["iter_counts"] = res["iter_counts"][:nd]
        res["loop_counts"] = {s: v[:nd] for s, v in res["loop_counts"].items()}
        res["sample_ticks"] = ticks[:nd]
        raise OracleBudget(res)
    return res


def run_fsm(kernel, target, m, n, seed, variant="plain", order=None, tick_chunk=100,
            tick_budget=None, x0=None, init_jitter=0.0, chain_offset=0, nthreads=1,
            surplus=True):
    """lockstep.py:308-416 restated (two-phase stop; see fsm_oracle.c).
    surplus=False skips the ticks chains take after their n-th sample (the
    engine's surplus=False; samples and per-sample counts are unchanged)."""
    ordp = None
    if order is not None:
        oa = (ctypes.c_int32 * len(order))(*order)
        ordp = ctypes.cast(oa, ctypes.POINTER(ctypes.c_int32))
    return _run(lib().or_run_fsm, kernel, target, m, n, seed, x0, init_jitter, chain_offset,
                nthreads, (VARIANTS[variant], ordp, int(tick_chunk), int(tick_budget or 0),
                           int(bool(surplus))))


def run_standard(kernel, target, m, n, seed, x0=None, init_jitter=0.0, chain_offset=0,
                 nthreads=1):
    """lockstep.py:238-305 restated."""
    return _run(lib().or_run_standard, kernel, target, m, n, seed, x0, init_jitter,
                chain_offset, nthreads, ())


def fill(seed, stream, counter, count, kind):
    out = np.empty(count, dtype=np.uint64 if kind == 0 else np.float64)
    lib().or_fill(seed & (2**64 - 1), stream & (2**64 - 1), counter & (2**64 - 1), count, kind,
                  out.ctypes.data)
    return out
