"""Freeze golden vectors from the LIVE reference (``/root/reference``).

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``fsm_mcmc`` in place and writes ``tests/golden/*.npz``.  The
fixtures pin the oracle (``oracle/``) and the CUDA path (``-m gpu`` tests).
New targets the reference lacks (Neal's funnel, the GP-classification
latent, the NaN-band fault target) are restated here as ``TargetModel``
closures, the way the reference's own tests build fake targets
(``pkg/tests/test_kernels.py:107``, ``pkg/tests/tests_common_conjugate.py:13``).
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, REF + "/src")
sys.path.insert(0, REF + "/tests")

from fsm_mcmc import prng  # noqa: E402
from fsm_mcmc.kernels import drmh_kernel, elliptical_kernel, nuts_kernel, slice_kernel  # noqa: E402
from fsm_mcmc.lockstep import (KernelRunError, TickBudgetExceeded,  # noqa: E402
                               init_batch, run_fsm_batched, run_standard_batched)
from fsm_mcmc.targets import (GaussianPriorDecomposition, TargetModel,  # noqa: E402
                              correlated_mog_target, equicorrelated_covariance,
                              gaussian_target, gp_hyperparameter_target,
                              make_synthetic_gp_dataset)
from tests_common_conjugate import conjugate_target  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
LOG_2PI = math.log(2.0 * math.pi)


# ---------------------------------------------------------------- new targets
def funnel_target(d: int, v_scale: float = 3.0) -> TargetModel:
    """Neal's funnel: v = x[0] ~ N(0, s^2); x[i] | v ~ N(0, e^v), i >= 1."""
    s = float(v_scale)

    def lp_grad(x):
        x = np.asarray(x, dtype=float)
        v = float(x[0])
        r = x[1:]
        ev = math.exp(-v)
        q = float(r @ r)
        lp = (-0.5 * (v / s) * (v / s) - math.log(s) - 0.5 * LOG_2PI
              - 0.5 * q * ev - 0.5 * (d - 1) * v - 0.5 * (d - 1) * LOG_2PI)
        g = np.empty(d)
        g[0] = -v / (s * s) + 0.5 * q * ev - 0.5 * (d - 1)
        g[1:] = -r * ev
        return lp, g

    return TargetModel(name=f"funnel-{d}d", dim=d, log_density=lambda x: lp_grad(x)[0],
                       gradient=lambda x: lp_grad(x)[1], log_density_and_grad=lp_grad)


def gp_class_data(n_pts: int, seed: int = 20240617):
    """Synthetic GP-classification latent problem."""
    rng = np.random.default_rng(seed)
    S = rng.normal(size=(n_pts, 2))
    sq = np.sum(S * S, axis=1)
    d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * (S @ S.T), 0.0)
    K = np.exp(-0.5 * d2) + 1e-6 * np.eye(n_pts)
    L = np.linalg.cholesky(K)
    f = L @ rng.normal(size=n_pts)
    y = np.where(rng.uniform(size=n_pts) < 1.0 / (1.0 + np.exp(-f)), 1.0, -1.0)
    return L, y


def gp_class_fspace_target(n_pts: int) -> TargetModel:
    L, y = gp_class_data(n_pts)
    return TargetModel(
        name=f"gpc-{n_pts}", dim=n_pts, log_density=lambda x: 0.0,
        gaussian_prior=GaussianPriorDecomposition(
            chol=L, residual_log_density=lambda x: float(-np.logaddexp(0.0, -y * x).sum())))


def logreg_data(n_obs: int, d: int, seed: int = 0):
    """Synthetic Bayesian logistic regression:
    X ~ N(0,1)/sqrt(d), theta* ~ N(0, I), y ~ Bernoulli(sigmoid(X theta*))."""
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n_obs, d)) / math.sqrt(d)
    theta = rng.normal(size=d)
    y = (rng.uniform(size=n_obs) < 1.0 / (1.0 + np.exp(-(X @ theta)))).astype(float)
    return X, y


def logreg_target(X, y) -> TargetModel:
    """log p(theta) = sum_i [y_i z_i - log(1 + e^{z_i})] - theta.theta/2, z = X theta;
    grad = X^T (y - sigmoid(z)) - theta."""
    d = X.shape[1]

    def lp_grad(theta):
        theta = np.asarray(theta, dtype=float)
        z = X @ theta
        lp = float(np.sum(y * z - np.logaddexp(0.0, z))) - 0.5 * float(theta @ theta)
        g = X.T @ (y - 1.0 / (1.0 + np.exp(-z))) - theta
        return lp, g

    return TargetModel(name=f"logreg-{X.shape[0]}x{d}", dim=d,
                       log_density=lambda t: lp_grad(t)[0], gradient=lambda t: lp_grad(t)[1],
                       log_density_and_grad=lp_grad)


def nan_band_target(d: int, threshold: float, value: float) -> TargetModel:
    """Standard normal that returns ``value`` (NaN or +inf) once x[0] > threshold."""
    def lp(x):
        x = np.asarray(x, dtype=float)
        if x[0] > threshold:
            return value
        return -0.5 * float(x @ x) - 0.5 * d * LOG_2PI
    return TargetModel(name="nanband", dim=d, log_density=lp)


def equicorr_gauss(d, rho):
    return gaussian_target(np.zeros(d), np.linalg.cholesky(equicorrelated_covariance(d, rho)))


# ------------------------------------------------------------------ helpers
def ledger_dict(prefix, samples, led, out):
    out[prefix + "samples"] = samples
    out[prefix + "iter_counts"] = led.iter_counts
    for s, mat in led.loop_exec_counts.items():
        out[prefix + f"loop_{s}"] = mat
    out[prefix + "tick_count"] = np.int64(led.tick_count)
    out[prefix + "block_exec_counts"] = led.block_exec_counts
    out[prefix + "charged_cost"] = np.float64(led.charged_cost)
    out[prefix + "native_shared_evals"] = np.int64(led.native_shared_evals)
    if led.sample_ticks is not None:
        out[prefix + "sample_ticks"] = led.sample_ticks


def run_case(name, bundle, target, m, n, seed, variants, extra=None, tick_chunk=100,
             standard=True, x0=None):
    out = {"m": np.int64(m), "n": np.int64(n), "seed": np.int64(seed),
           "tick_chunk": np.int64(tick_chunk)}
    if x0 is not None:
        out["x0"] = np.asarray(x0, dtype=float)
    if extra:
        out.update(extra)
    for v in variants:
        s, led = run_fsm_batched(bundle, target, init_batch(bundle, target, m, seed, x0=x0), n,
                                 step_variant=v, record_sample_ticks=True,
                                 tick_chunk=tick_chunk)
        ledger_dict(f"{v}_", s, led, out)
    if standard:
        s, led = run_standard_batched(bundle, target, init_batch(bundle, target, m, seed, x0=x0), n)
        ledger_dict("standard_", s, led, out)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print("wrote", name, {k: getattr(v, "shape", ()) for k, v in out.items() if "samples" in k})


def prng_golden():
    out = {}
    trip = [(0, 0, 0), (123, 4, 567), (7, 1, 0), (2**64 - 1, 2**63 + 5, 2**64 - 3),
            (99, 12345, 10**12), (2024, 0, 0)]
    bits = [prng._bits(*t) for t in trip]
    out["trip"] = np.array(trip, dtype=np.uint64)
    out["bits"] = np.array(bits, dtype=np.uint64)
    out["uniform"] = np.array([prng.uniform(prng.key(*t))[0] for t in trip])
    out["normal"] = np.array([prng.normal(prng.key(*t))[0] for t in trip])
    kids = prng.split(prng.key(0), 3) + prng.split(prng.key(7, 99), 5)
    out["split_streams"] = np.array([k.stream for k in kids], dtype=np.uint64)
    # long runs of draws on a few chain streams (covers both ndtri branches)
    keys = prng.split(prng.key(5), 4)
    N = 4096
    out["run_streams"] = np.array([k.stream for k in keys], dtype=np.uint64)
    out["run_uniform"] = np.stack([prng.uniform_block(k, N)[0] for k in keys])
    out["run_normal"] = np.stack([prng.normal_vec(k, N)[0] for k in keys])
    # chain 1 of seed 7
    k1 = prng.split(prng.key(7), 2)[1]
    out["seed7_chain1_normal"] = np.float64(prng.normal(k1)[0])
    out["seed7_chain1_uniform"] = np.float64(prng.uniform(k1)[0])
    np.savez_compressed(os.path.join(OUT, "prng.npz"), **out)
    print("wrote prng")


def error_golden():
    out = {}
    t = nan_band_target(2, 2.8, math.nan)
    b = drmh_kernel(5, 1.0)
    for v in ("plain", "bundled"):
        try:
            run_fsm_batched(b, t, init_batch(b, t, 6, 3), 400, step_variant=v)
            raise SystemExit("expected a failure")
        except KernelRunError as e:
            out[f"nan_{v}"] = np.array([e.chain, e.iteration])
            out[f"nan_{v}_label"] = np.array(e.cause.label)
    t = nan_band_target(2, 2.8, math.inf)
    try:
        run_standard_batched(b, t, init_batch(b, t, 6, 3), 400)
        raise SystemExit("expected a failure")
    except KernelRunError as e:
        out["inf_standard"] = np.array([e.chain, e.iteration])
        out["inf_standard_label"] = np.array(e.cause.label)
    tn = gaussian_target(np.zeros(1), np.eye(1))
    b = drmh_kernel(10, 0.5)
    try:
        run_fsm_batched(b, tn, init_batch(b, tn, 2, 7), 10_000, tick_budget=250)
        raise SystemExit("expected budget overrun")
    except TickBudgetExceeded as e:
        out["budget_tick_count"] = np.int64(e.ledger.tick_count)
        out["budget_sample_counts"] = np.array(e.sample_counts)
        out["budget_iter_counts"] = e.ledger.iter_counts
    np.savez_compressed(os.path.join(OUT, "errors.npz"), **out)
    print("wrote errors")


def main():
    prng_golden()
    error_golden()
    # DRMH ------------------------------------------------------------
    run_case("drmh_mog10", drmh_kernel(100, 0.1), correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0]),
             m=16, n=120, seed=0, variants=("plain", "bundled", "amortized"))
    run_case("drmh_funnel10", drmh_kernel(100, 0.1), funnel_target(10),
             m=16, n=120, seed=1, variants=("plain", "bundled"))
    run_case("drmh_std1", drmh_kernel(100, 0.1), gaussian_target(np.zeros(1), np.eye(1)),
             m=8, n=200, seed=2, variants=("plain", "bundled"), tick_chunk=1)
    run_case("drmh_gauss3", drmh_kernel(20, 0.7),
             gaussian_target(np.array([0.5, -1.0, 2.0]),
                             np.array([[1.0, 0, 0], [0.3, 0.8, 0], [-0.2, 0.1, 0.5]])),
             m=8, n=150, seed=3, variants=("plain", "bundled"), tick_chunk=7)
    # ESS -------------------------------------------------------------
    run_case("ess_conj100", elliptical_kernel(), conjugate_target(dim=100),
             m=8, n=100, seed=0, variants=("plain", "bundled", "amortized"))
    run_case("ess_conj2", elliptical_kernel(), conjugate_target(dim=2),
             m=8, n=200, seed=4, variants=("plain", "bundled"), tick_chunk=1)
    L, y = gp_class_data(64)
    run_case("ess_gpc64", elliptical_kernel(), gp_class_fspace_target(64),
             m=6, n=60, seed=5, variants=("amortized", "bundled"),
             extra={"L": L, "y": y})
    # NUTS ------------------------------------------------------------
    run_case("nuts_corr100", nuts_kernel(0.05, 10), equicorr_gauss(100, 0.99),
             m=6, n=40, seed=0, variants=("plain", "bundled"))
    run_case("nuts_mog10", nuts_kernel(0.2, 6), correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0]),
             m=8, n=60, seed=6, variants=("plain", "bundled"), tick_chunk=10)
    run_case("nuts_funnel5", nuts_kernel(0.3, 5, divergence_threshold=50.0), funnel_target(5),
             m=8, n=60, seed=7, variants=("plain", "bundled"))
    run_case("nuts_std2", nuts_kernel(0.9, 4), gaussian_target(np.zeros(2), np.eye(2)),
             m=8, n=100, seed=8, variants=("plain", "bundled"), tick_chunk=1)
    X, y = logreg_data(512, 16, seed=0)
    run_case("nuts_logreg512x16", nuts_kernel(0.1, 8), logreg_target(X, y),
             m=6, n=40, seed=9, variants=("plain", "bundled"), extra={"X": X, "y": y})
    main_split_only()
    main_slice_only()
    main_efficiency_only()
    main_gp_only()
    main_cli_only()


def main_split_only():
    run_case("drmh_split_std1", drmh_kernel(50, 0.4, split_body=True),
             gaussian_target(np.zeros(1), np.eye(1)), m=6, n=80, seed=5,
             variants=("plain", "bundled"), tick_chunk=1)
    run_case("drmh_split_mog10", drmh_kernel(100, 0.1, split_body=True),
             correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0]), m=8, n=40, seed=6,
             variants=("plain", "bundled"))


def main_slice_only():
    """The univariate slice sampler (slice_sampling.py): stepping-out and
    shrinkage counts, the expansion cap, compact support, and failures."""
    std1 = gaussian_target(np.zeros(1), np.eye(1))
    run_case("slice_std1", slice_kernel(1.0), std1, m=8, n=200, seed=10,
             variants=("plain", "bundled", "amortized"), tick_chunk=1)
    run_case("slice_narrow", slice_kernel(0.2, max_expansions=50),
             gaussian_target(np.array([1.5]), np.array([[2.0]])), m=6, n=120, seed=11,
             variants=("plain", "bundled"), tick_chunk=10)
    run_case("slice_cap", slice_kernel(0.05, max_expansions=3), std1, m=6, n=100, seed=12,
             variants=("plain", "bundled"))

    def uniform01(x):
        return 0.0 if 0.0 <= float(x[0]) <= 1.0 else -math.inf
    box = TargetModel(name="uniform01", dim=1, log_density=uniform01)
    run_case("slice_box", slice_kernel(10.0, max_expansions=8), box, m=4, n=200, seed=9,
             variants=("plain", "bundled"), x0=np.array([0.5]))
    out = {}
    t = nan_band_target(1, 2.0, math.nan)
    b = slice_kernel(1.0)
    for v in ("plain", "bundled"):
        try:
            run_fsm_batched(b, t, init_batch(b, t, 6, 3), 400, step_variant=v)
            raise SystemExit("expected a failure")
        except KernelRunError as e:
            out[f"nan_{v}"] = np.array([e.chain, e.iteration])
            out[f"nan_{v}_label"] = np.array(e.cause.label)
    try:
        run_standard_batched(b, t, init_batch(b, t, 6, 3), 400)
        raise SystemExit("expected a failure")
    except KernelRunError as e:
        out["nan_standard"] = np.array([e.chain, e.iteration])
        out["nan_standard_label"] = np.array(e.cause.label)
    np.savez_compressed(os.path.join(OUT, "errors_slice.npz"), **out)
    print("wrote errors_slice", out)


def main_gp_only():
    """The GP-hyperparameter posterior (targets.py:191-265; the paper's section
    7.2 workload) under all three multivariate kernels."""
    X, y = make_synthetic_gp_dataset(50, 3)
    t = gp_hyperparameter_target(X, y)
    ex = {"X": X, "y": y}
    x0 = np.array([0.3, 1.0, 1.0])
    run_case("ess_gp50", elliptical_kernel(), t, m=6, n=60, seed=13,
             variants=("amortized", "bundled"), extra=ex, x0=x0)
    run_case("drmh_gp50", drmh_kernel(20, 0.2), t, m=6, n=60, seed=14,
             variants=("plain", "bundled"), extra=ex, x0=x0)
    run_case("nuts_gp50", nuts_kernel(0.1, 6), t, m=4, n=25, seed=15,
             variants=("plain", "bundled"), extra=ex, x0=x0)


CLI_CONFIGS = [
    dict(kernel="drmh", target="std-normal", dim=2, chains=16, samples=200, variant="bundled",
         seeds=(0, 1)),
    dict(kernel="slice", target="std-normal", dim=1, chains=8, samples=150, variant="plain",
         seeds=(3,)),
    dict(kernel="nuts", target="gaussian-corr", dim=5, chains=6, samples=60, variant="bundled",
         target_rho=0.9, seeds=(2,)),
    dict(kernel="elliptical", target="gp-synthetic", chains=4, samples=40, variant="amortized",
         seeds=(5,)),
    dict(kernel="drmh", target="mog", dim=4, chains=12, samples=100, variant="plain",
         drmh_split_body=True, target_rho=0.5, seeds=(7,)),
]


def main_cli_only():
    """cli.py run_experiment rows (write=False) and config validation/hashes."""
    import json
    from fsm_mcmc import cli
    out = {"runs": [], "validate": [], "hash_default": cli.RunConfig().config_hash()}
    for kw in CLI_CONFIGS:
        res = cli.run_experiment(cli.RunConfig(**kw), write=False)
        out["runs"].append({"config": {k: list(v) if isinstance(v, tuple) else v
                                       for k, v in kw.items()},
                            "hash": res.config.config_hash(), "rows": res.rows})
    for kw in (dict(kernel="slice", target="std-normal", dim=3), dict(kernel="elliptical"),
               dict(kernel="bogus", chains=0, samples=0, variant="x", seeds=()),
               dict(target="mog", target_rho=1.5, tick_budget=0, dim=0),
               dict(kernel="nuts", nuts_step_size=-1.0, nuts_max_depth=0),
               dict(kernel="drmh", drmh_max_tries=0, drmh_proposal_scale=0.0)):
        out["validate"].append({"config": kw, "errors": cli.RunConfig(**kw).validate()})
    with open(os.path.join(OUT, "cli.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote cli")


def main_efficiency_only():
    """Cost-theory analytics (analysis.py:53-324) on fixed inputs."""
    from fsm_mcmc import analysis as A
    from fsm_mcmc.lockstep import CostParams
    out = {}
    rng = np.random.default_rng(77)
    N = rng.geometric(0.2, size=(300, 64)).astype(np.int64)
    out["N"] = N
    out["barrier"] = np.float64(A.barrier_cost(N))
    out["desync"] = np.float64(A.desync_cost(N))
    params = CostParams(block_costs=(0.05, 1.0, 0.05), alpha=1.0, loop_states=(2,))
    rep = A.efficiency_report(params, N, standard_cost_per_sample=3.0, fsm_cost_per_sample=1.5)
    out["report"] = np.array([rep.m, rep.E_of_m, rep.R_of_m, rep.mean_N, rep.mean_max_N])
    for m in (1, 16, 1024):
        b = A.bound_R(m, samples=N.reshape(-1), n_replicates=2000, seed=5)
        out[f"bound_{m}"] = np.array([b.estimate, b.std_error])
    b = A.bound_R(16, bernoulli=(0.1, 3.0), n_replicates=20_000, seed=1)
    out["bound_bern"] = np.array([b.estimate, b.std_error, b.closed_form])
    rep = A.verify_prop_bound(500, seed=3)
    out["prop"] = np.array([len(rep.violations), rep.tightness_cases, rep.tightness_max_rel_err,
                            rep.max_excess])
    runs = [rng.geometric(0.4, size=(4000, 8)) for _ in range(6)]
    out["conc_runs"] = np.stack(runs)
    c = A.concentration_check(runs, (10, 100, 1000, 4000), params)
    out["conc"] = np.array([c.slope, c.slope_stderr, c.limit_estimate, *c.deviations])
    np.savez_compressed(os.path.join(OUT, "efficiency.npz"), **out)
    print("wrote efficiency")


def main_logreg_only():
    X, y = logreg_data(512, 16, seed=0)
    run_case("nuts_logreg512x16", nuts_kernel(0.1, 8), logreg_target(X, y),
             m=6, n=40, seed=9, variants=("plain", "bundled"), extra={"X": X, "y": y})


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "logreg":
        main_logreg_only()
    elif len(sys.argv) > 1 and sys.argv[1] == "split":
        main_split_only()
    elif len(sys.argv) > 1 and sys.argv[1] == "slice":
        main_slice_only()
    elif len(sys.argv) > 1 and sys.argv[1] == "efficiency":
        main_efficiency_only()
    elif len(sys.argv) > 1 and sys.argv[1] == "gp":
        main_gp_only()
    elif len(sys.argv) > 1 and sys.argv[1] == "cli":
        main_cli_only()
    else:
        main()
