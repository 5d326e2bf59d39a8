"""Batched evaluators for dense-contraction targets (BASELINE configs 4-5).

In batched-evaluation mode (``run_fsm_batched(..., evaluator=...)``) every
chain advances to its next log-density request and all requests of a round
are evaluated together, so a dense target becomes a pair of contractions
across chains instead of one GEMV per chain (the paper's amortized step,
``fsm.py:252-273``).

Bayesian logistic regression (``targets.logistic_regression_target``):

    Z = Θ Xᵀ                       [k, N]   (k requesting chains)
    lp_j = Σ_i y_i z_ji − log(1 + e^{z_ji}) − θ_j·θ_j / 2
    G = (y − σ(Z)) X − Θ           [k, d]

``precision="fp64"`` evaluates in IEEE double (parity with the per-chain
plugin up to reduction order).  ``"tf32"`` runs both contractions as cuBLAS
TF32 GEMMs with the σ / softplus / row-sum epilogue in one pass over Z
(``fsmc_logreg_epilogue``).  ``"bf16-tc"`` / ``"fp16-tc"`` are the fused
hand-written tcgen05 kernel (``csrc/logreg_tc.cu``, d = 256): 16-bit operands
by TMA, both products accumulated in fp32 in TMEM, the logits never stored.
fp16 carries 11 mantissa bits to bf16's 8 at the same tensor rate, so theta
is rounded 8x more finely: at N = 100k the log density is the sum of 1e5
terms, and its error from rounding theta scales with N (tests/
test_gpu_distribution.py).  The reduced precisions give distributional
parity only.  Chains are processed in tiles so a
materialised Z never exceeds ``tile`` rows.
"""

from __future__ import annotations

import torch

from . import _lib

__all__ = ["LogisticRegressionEvaluator"]


class LogisticRegressionEvaluator:
    def __init__(self, X, y, precision: str = "fp64", tile: int = 4096):
        if precision not in ("fp64", "tf32", "bf16-tc", "fp16-tc"):
            raise ValueError("precision must be fp64, tf32, bf16-tc or fp16-tc")
        self.precision = precision
        self.tile = int(tile)
        X = torch.as_tensor(X, dtype=torch.float64, device="cuda").contiguous()
        y = torch.as_tensor(y, dtype=torch.float64, device="cuda").contiguous()
        if precision == "fp64":
            self.X, self.y = X, y
        elif precision == "tf32":
            self.X, self.y = X.to(torch.float32), y.to(torch.float32)
            self.XT = self.X.T.contiguous()
        else:
            n, d = X.shape
            if d != 256 or n % 8:
                raise ValueError("the fused kernel needs d = 256 and n_obs a multiple of 8")
            self.n_obs, self.d = n, d
            self.h16 = torch.float16 if precision == "fp16-tc" else torch.bfloat16
            self.operand = 1 if precision == "fp16-tc" else 0
            self.Xb = X.to(self.h16).contiguous()
            self.XTb = self.Xb.T.contiguous()
            self.xty = (X.T @ y).contiguous()     # label terms, linear in theta (fp64)
            self.theta_b = torch.empty(0, dtype=self.h16, device="cuda")

    def __call__(self, theta: torch.Tensor, lp: torch.Tensor, grad: torch.Tensor | None):
        if self.precision == "fp64":
            return self._fp64(theta, lp, grad)
        if self.precision in ("bf16-tc", "fp16-tc"):
            return self._fused(theta, lp, grad)
        k = theta.shape[0]
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        try:
            for lo in range(0, k, self.tile):
                hi = min(k, lo + self.tile)
                th = theta[lo:hi]
                z = th.to(torch.float32) @ self.XT                      # [t, N] fp32
                lp[lo:hi] = -0.5 * (th * th).sum(dim=1)
                _lib.check(_lib.lib().fsmc_logreg_epilogue(
                    z.data_ptr(), self.y.data_ptr(), hi - lo, z.shape[1], z.data_ptr(),
                    lp[lo:hi].data_ptr(), _lib.stream_ptr()), "fsmc_logreg_epilogue")
                if grad is not None:
                    grad[lo:hi] = (z @ self.X).to(torch.float64) - th
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev

    def _fp64(self, theta, lp, grad):
        k = theta.shape[0]
        for lo in range(0, k, self.tile):
            hi = min(k, lo + self.tile)
            th = theta[lo:hi]
            z = th @ self.X.T
            sp = torch.clamp_min(z, 0) + torch.log1p(torch.exp(-z.abs()))
            lp[lo:hi] = (self.y * z - sp).sum(dim=1) - 0.5 * (th * th).sum(dim=1)
            if grad is not None:
                grad[lo:hi] = (self.y - torch.sigmoid(z)) @ self.X - th

    def _fused(self, theta, lp, grad):
        k = theta.shape[0]
        need = -(-k // 128) * 128 * self.d
        if self.theta_b.numel() < need:
            self.theta_b = torch.empty(need, dtype=self.h16, device="cuda")
        g = grad if grad is not None else torch.empty((k, self.d), dtype=torch.float64, device="cuda")
        th = theta.contiguous()
        st = _lib.lib().fsmc_logreg_tc_eval2(th.data_ptr(), k, self.theta_b.data_ptr(),
                                             self.Xb.data_ptr(), self.XTb.data_ptr(),
                                             self.xty.data_ptr(), self.n_obs, self.d, lp.data_ptr(),
                                             g.data_ptr(), self.operand, _lib.stream_ptr())
        if st != 0:
            raise RuntimeError("fsmc_logreg_tc_eval: " +
                               _lib.lib().fsmc_logreg_tc_last_error().decode())


# ---------------------------------------------------------------- prior transform
# Elliptical slice sampling with a dense Gaussian prior draws nu = L eps at
# every INIT (elliptical.py:73).  In fsmc_advance_prior mode the parked eps
# rows of a round are transformed together: one triangular matrix product
# across chains (cuBLAS DTRMM, d^2 flops per row instead of a GEMV per chain).
_CUBLAS = None


def _cublas():
    global _CUBLAS
    if _CUBLAS is None:
        import ctypes
        import os

        import nvidia.cublas as nc
        lib = ctypes.CDLL(os.path.join(list(nc.__path__)[0], "lib", "libcublas.so.12"))
        P = ctypes.c_void_p
        lib.cublasDtrmm_v2.restype = ctypes.c_int
        lib.cublasDtrmm_v2.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                       P, ctypes.c_int, P, ctypes.c_int, P, ctypes.c_int]
        _CUBLAS = lib
    return _CUBLAS


class PriorTransform:
    """nu[r] = L nu[r] for the rows of a round, L lower-triangular (the
    target's prior factor; ``Lt`` = Lᵀ row-major = L column-major).
    ``method="dmma"``: the hand-written fp64 tensor-core triangular product
    (``fsmc_prior_trmm``, csrc/prior_trmm.cu); ``"trmm"``: cuBLAS DTRMM
    (half the flops of a dense product); ``"gemm"``: a dense DGEMM
    ``rows @ Lᵀ``."""

    def __init__(self, Lt: torch.Tensor, method: str = "dmma", target=None):
        if method not in ("dmma", "trmm", "gemm"):
            raise ValueError("method must be dmma, trmm or gemm")
        if method == "dmma" and target is None:
            raise ValueError("the dmma transform needs the target (its device descriptor)")
        self.Lt, self.method, self.d = Lt, method, Lt.shape[0]
        self.tgt = target.struct() if target is not None else None
        self.tmp = None
        self.one = None

    def __call__(self, rows: torch.Tensor) -> None:
        k, d = rows.shape
        if self.tmp is None or self.tmp.shape[0] < k:
            self.tmp = torch.empty_like(rows)
        out = self.tmp[:k]
        if self.method == "dmma":
            import ctypes
            st = _lib.lib().fsmc_prior_trmm(ctypes.byref(self.tgt), rows.data_ptr(), out.data_ptr(),
                                            k, _lib.stream_ptr())
            if st != 0:
                raise _lib.EngineError("fsmc_prior_trmm: " +
                                       _lib.lib().fsmc_prior_trmm_last_error().decode())
            return
        if self.method == "gemm":
            torch.mm(rows, self.Lt, out=out)
        else:
            import ctypes
            if self.one is None:
                self.one = ctypes.c_double(1.0)
            h = torch.cuda.current_blas_handle()     # bound to the current stream
            # column-major: C (d x k) = L (d x d, lower) * B (d x k); B = rows
            st = _cublas().cublasDtrmm_v2(h, 0, 0, 0, 0, d, k, ctypes.byref(self.one),
                                          self.Lt.data_ptr(), d, rows.data_ptr(), d,
                                          out.data_ptr(), d)
            if st != 0:
                raise RuntimeError(f"cublasDtrmm failed ({st})")
        rows.copy_(out)


# ----------------------------------------------------------- GP hyperparameters
_LOG_2PI = 1.8378770664093453
_FAILURE = torch.tensor([0x7ff80000dead0001], dtype=torch.int64).view(torch.float64)  # fsm_device.cuh


class GPHyperEvaluator:
    """Batched evaluator of the GP-hyperparameter target (targets.py:191-265)
    for designs too large for the per-chain shared-memory plugin (the
    paper's section 7.2 uses n = 414 observations).  Per round, for the k
    requesting chains theta = (sigma, tau, lam):

        K_j = tau_j^2 exp(-lam_j^2 D2) + (sigma_j^2 + jitter) I     [k, n, n]
        L_j = chol(K_j),  alpha_j = K_j^-1 y,  lml_j = -y.alpha_j/2 - sum log diag L_j - n log(2 pi)/2

    by ``fsmc_gp_lml_grad`` (csrc/gp_chol.cu: one CTA per chain, a
    left-looking blocked Cholesky with K formed on the fly; with the
    gradient, alpha = K^-1 y, W = L^-1 and the trace terms from the same
    factor).  ``torch_eval`` (batched torch.linalg factorizations) is kept as
    a cross-check and for single-request value rounds, which one matrix
    spread over the whole GPU serves faster.  ``residual=True`` returns the marginal likelihood (the
    elliptical kernel's residual log density); otherwise the N(0, I) prior
    terms are added.  The gradient is the reference's trace form with
    A = alpha alpha^T - K^-1.  A kernel matrix that is not positive definite
    returns the plugin's TargetError payload for that chain."""

    def __init__(self, d2, y, jitter: float, residual: bool, tile: int = 512):
        self.d2 = torch.as_tensor(d2, dtype=torch.float64, device="cuda").contiguous()
        self.y = torch.as_tensor(y, dtype=torch.float64, device="cuda").contiguous()
        self.jitter, self.residual, self.tile = float(jitter), bool(residual), int(tile)
        self.n = self.y.shape[0]
        self.slots = torch.cuda.get_device_properties(self.d2.device).multi_processor_count
        self.work = None
        self.min_kernel_rows = 16

    def __call__(self, theta, lp, g=None):
        # the hand-written kernel (csrc/gp_chol.cu, one CTA per chain) for every
        # gradient round and for value rounds with enough requests to fill the
        # SMs; a handful of value requests runs faster through the library
        # factorization, which spreads one matrix over the whole GPU
        if self.n > _lib.lib().fsmc_gp_lml_max_rows():
            return self.torch_eval(theta, lp, g)
        if g is None and theta.shape[0] < self.min_kernel_rows:
            return self.torch_eval(theta, lp, g)
        if self.work is None:
            self.work = torch.empty((self.slots, self.n, self.n), dtype=torch.float64,
                                    device=self.d2.device)
        theta = theta.contiguous()
        st = _lib.lib().fsmc_gp_lml_grad(theta.data_ptr(), theta.shape[0], self.d2.data_ptr(),
                                         self.y.data_ptr(), self.n, self.jitter, int(self.residual),
                                         self.work.data_ptr(), self.slots, lp.data_ptr(),
                                         _lib.ptr(g), _lib.stream_ptr())
        if st != 0:
            raise _lib.EngineError(_lib.lib().fsmc_gp_last_error().decode())

    def torch_eval(self, theta, lp, g=None):
        """Value (and gradient) through torch.linalg's batched factorizations
        (the gradient path: it needs K^-1 for the trace terms)."""
        n, d2, y = self.n, self.d2, self.y
        fail = _FAILURE.to(lp.device)
        for a in range(0, theta.shape[0], self.tile):
            th = theta[a:a + self.tile]
            s, t, lam = th[:, 0], th[:, 1], th[:, 2]
            E = torch.exp((-(lam * lam))[:, None, None] * d2)
            K = (t * t)[:, None, None] * E
            K.diagonal(dim1=1, dim2=2).add_((s * s + self.jitter)[:, None])
            L, info = torch.linalg.cholesky_ex(K)
            alpha = torch.cholesky_solve(y.expand(th.shape[0], n)[..., None], L)[..., 0]
            logdet = 2.0 * torch.log(L.diagonal(dim1=1, dim2=2)).sum(-1)
            out = -0.5 * (y * alpha).sum(-1) - 0.5 * logdet - 0.5 * n * _LOG_2PI
            if not self.residual:
                out = out - 0.5 * (th * th).sum(-1) - 1.5 * _LOG_2PI
            bad = info != 0
            lp[a:a + self.tile] = torch.where(bad, fail, out)
            if g is not None:
                A = alpha[:, :, None] * alpha[:, None, :] - torch.cholesky_inverse(L)
                AE = A * E
                gr = torch.stack([s * A.diagonal(dim1=1, dim2=2).sum(-1), t * AE.sum((1, 2)),
                                  -lam * t * t * (AE * d2).sum((1, 2))], dim=1)
                if not self.residual:
                    gr = gr - th
                g[a:a + self.tile] = gr
