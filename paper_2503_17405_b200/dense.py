"""Batched evaluators for dense-contraction targets (BASELINE configs 4-5).

In batched-evaluation mode (``run_fsm_batched(..., evaluator=...)``) every
chain advances to its next log-density request and all requests of a round
are evaluated together, so a dense target becomes a pair of GEMMs across
chains instead of one GEMV per chain (the paper's amortized step,
``fsm.py:252-273``).

Bayesian logistic regression (``targets.logistic_regression_target``):

    Z = Θ Xᵀ                       [k, N]   (k requesting chains)
    lp_j = Σ_i y_i z_ji − log(1 + e^{z_ji}) − θ_j·θ_j / 2
    G = (y − σ(Z)) X − Θ           [k, d]

``precision="fp64"`` evaluates in IEEE double (parity with the per-chain
plugin to reduction order); ``"tf32"`` / ``"bf16"`` run the contractions on
the tensor cores with fp32 accumulation (distributional parity only).
Chains are processed in tiles so Z never exceeds ``tile`` rows.
"""

from __future__ import annotations

import torch

__all__ = ["LogisticRegressionEvaluator"]


class LogisticRegressionEvaluator:
    def __init__(self, X, y, precision: str = "fp64", tile: int = 4096):
        if precision not in ("fp64", "tf32", "bf16", "fp32"):
            raise ValueError("precision must be fp64, fp32, tf32 or bf16")
        self.precision = precision
        self.tile = int(tile)
        X = torch.as_tensor(X, dtype=torch.float64, device="cuda").contiguous()
        y = torch.as_tensor(y, dtype=torch.float64, device="cuda").contiguous()
        if precision == "fp64":
            self.X, self.y = X, y
        elif precision == "bf16":
            self.X, self.y = X.to(torch.bfloat16), y.to(torch.float32)
        else:
            self.X, self.y = X.to(torch.float32), y.to(torch.float32)

    def __call__(self, theta: torch.Tensor, lp: torch.Tensor, grad: torch.Tensor | None):
        k = theta.shape[0]
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = self.precision == "tf32"
        try:
            for lo in range(0, k, self.tile):
                hi = min(k, lo + self.tile)
                th = theta[lo:hi]
                tc = th.to(self.X.dtype)
                z = tc @ self.X.T                                   # [t, N]
                zf = z.to(self.y.dtype)
                # numpy logaddexp(0, z) = max(z, 0) + log1p(exp(-|z|))
                sp = torch.clamp_min(zf, 0) + torch.log1p(torch.exp(-zf.abs()))
                lp[lo:hi] = ((self.y * zf - sp).sum(dim=1)).to(torch.float64) \
                    - 0.5 * (th * th).sum(dim=1)
                if grad is not None:
                    r = (self.y - torch.sigmoid(zf)).to(self.X.dtype)
                    grad[lo:hi] = (r @ self.X).to(torch.float64) - th
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
