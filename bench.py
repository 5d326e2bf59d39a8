"""bench.py -- samples/sec and ESS/sec of the FSM engine (BASELINE.json metric).

One *step* = one complete multi-chain sampling job through the public API:
init_batch(m chains) + run_fsm_batched(n samples per chain) on the device,
inputs resident in HBM.  Default workload = BASELINE config 2 (the metric's
single-GPU config): DRMH (M=100, scale 0.1) on the 10-d correlated MoG
(rho=0.9, modes -3/0/3), m=65536 chains, n=1000, bundled executor.

Under torchrun each rank owns m chains (weak scaling, chain offset rank*m,
no data-path collective); ESS/R-hat partials are all-reduced over NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4] [--impl reference]

--impl reference times the CPU oracle (oracle/, a C port of the reference's
path) on this host's cores for the same metric/config (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

# large per-step outputs (samples [n][m][d]) are reallocated every step: keep
# the caching allocator from fragmenting into fresh cudaMalloc/cudaFree calls
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec & ESS/sec at m chains (1/2/4/8 B200); speed-up vs lock-step vmap"
# executed fp64 flops per DRMH proposal on the MoG d=10 target (ncu SASS op
# counts, DFMA counted twice: generator 65.1 per draw x 11 + step kernel 260)
FP64_FLOPS_PER_PROPOSAL = 976.0
# ncu instruction counts of the C2 kernel pair (tools/gpujobs/r05_w.sh)
ISSUE_PROFILE = "r05_c2_issue.json"

CONFIGS = {
    "c2": dict(workload="C2: DRMH FSM, correlated MoG d=10 (rho=0.9, modes -3/0/3), M=100, "
                        "scale=0.1, bundled", family="drmh", m=65536, n=1000, d=10,
               variant="bundled", m_cpu=256, draw_window=4070, draw_parts=8),
    "c1": dict(workload="C1: elliptical slice FSM, conjugate Gaussian-likelihood d=100, amortized",
               family="ess", m=128, n=1000, d=100, variant="amortized", m_cpu=32, lanes=128),
    "c3": dict(workload="C3: NUTS FSM, equicorrelated Gaussian d=100 rho=0.99, eps=0.05, depth 10",
               family="nuts", m=16384, n=1000, d=100, variant="bundled", m_cpu=16),
    "c4": dict(workload="C4: elliptical slice FSM, GP-classification latent d=1024 (f-space)",
               family="ess", m=8192, n=200, d=1024, variant="amortized", m_cpu=4,
               prior_transform="dmma", prior_parts=3),
    # the fp32 throughput mode on configs 2 and 3 (separate lines, never the headline)
    "c2f": dict(workload="C2 in the fp32 throughput mode: DRMH FSM, correlated MoG d=10 (rho=0.9, "
                         "modes -3/0/3), M=100, scale=0.1, bundled; fp32 state and arithmetic, "
                         "fp64 reference draws rounded once; distributional parity only",
                family="drmh", m=65536, n=1000, d=10, variant="bundled", m_cpu=256,
                draw_window=4070, draw_parts=8, precision="fp32"),
    "c3f": dict(workload="C3 in the fp32 throughput mode: NUTS FSM, equicorrelated Gaussian d=100 "
                         "rho=0.99, eps=0.05, depth 10; fp32 state and arithmetic; distributional "
                         "parity only",
                family="nuts", m=16384, n=1000, d=100, variant="bundled", m_cpu=16,
                precision="fp32"),
    "c5": dict(workload="C5: NUTS FSM, Bayesian logistic regression N=100k d=256, eps=0.01, "
                        "depth 10; fp64 chain state, log density and gradient by the fused "
                        "tcgen05 kernel across chains (fp16 operands, fp32 accumulation; "
                        "distributional parity: profiles/r04_c5_distribution.json)",
               family="nuts", m=131072, n=32, d=256, variant="bundled", m_cpu=16, n_cpu=2, n_obs=100_000,
               batched="fp16-tc"),
}


# arithmetic of the line: fp64 everywhere unless a reduced-precision batched
# evaluator computes the log density and gradient
EVAL_DTYPE = {"bf16-tc": "f64 state / bf16 evaluator (fp32 accumulate)",
              "fp16-tc": "f64 state / fp16 evaluator (fp32 accumulate)",
              "tf32-tc": "f64 state / tf32 evaluator (fp32 accumulate)",
              "tf32": "f64 state / tf32 evaluator (cuBLAS)"}

_LOGREG = {}


def logreg_data(cfg):
    key = (cfg["n_obs"], cfg["d"])
    if key not in _LOGREG:
        from paper_2503_17405_b200.targets import logistic_regression_data
        _LOGREG[key] = logistic_regression_data(cfg["n_obs"], cfg["d"], seed=0)
    return _LOGREG[key]


def make_workload(cfg, fm=None, oracle=False):
    """Kernel + target of a config, for the engine or for the oracle."""
    if cfg.get("n_obs"):
        X, y = logreg_data(cfg)
        if oracle:
            from oracle import oracle as O
            return O.nuts(0.01, 10), O.logreg(X, y)
        return fm.nuts_kernel(0.01, 10), fm.targets.logistic_regression_target(X, y)
    if oracle:
        from oracle import oracle as O
        if cfg["family"] == "drmh":
            return O.drmh(100, 0.1), O.mog(10, 0.9, [-3.0, 0.0, 3.0])
        if cfg["family"] == "nuts":
            return O.nuts(0.05, 10), O.gaussian(np.zeros(100), np.linalg.cholesky(
                O.equicorrelated_covariance(100, 0.99)))
        if cfg["d"] == 100:
            return O.elliptical(), O.conjugate(100)
        from paper_2503_17405_b200.targets import gp_classification_data
        L, y = gp_classification_data(cfg["d"])
        return O.elliptical(), O.logistic_fspace(L, y)
    if cfg["family"] == "drmh":
        return fm.drmh_kernel(100, 0.1), fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
    if cfg["family"] == "nuts":
        return fm.nuts_kernel(0.05, 10), fm.equicorrelated_gaussian_target(100, 0.99)
    if cfg["d"] == 100:
        return fm.elliptical_kernel(), fm.conjugate_target(100)
    return fm.elliptical_kernel(), fm.gp_classification_target(cfg["d"])


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        self.q, self.index = q, index
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        # sampling is live before the timed region starts (nvidia-smi takes a
        # while to produce its first row)
        t0 = time.time()
        while self.p is not None and time.time() - t0 < 5.0:
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.01)
        self.skip = 0
        if self.p is not None:
            with open(self.f.name) as g:
                self.skip = len([r for r in g.read().splitlines() if r.strip()])

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        rows = rows[self.skip:]          # rows written before the timed region began
        if not rows:                     # a region shorter than the interval: one row right after it
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=20).stdout
                rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
            except (OSError, subprocess.SubprocessError):
                rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[4:8]):
                    if v.strip() == "Active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU oracle
def cpu_baseline(cfg, steps=1, warmup=0, seed=0):
    """The oracle (C port of the reference's path) on all host cores, on a
    bounded sample of the workload: m_cpu chains x n samples per step."""
    from oracle import oracle as O
    kern, targ = make_workload(cfg, oracle=True)
    threads = os.cpu_count() or 1
    m_cpu, n = cfg["m_cpu"], cfg.get("n_cpu", cfg["n"])
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        # surplus ticks skipped, as the engine's timed runs skip them (surplus=False)
        O.run_fsm(kern, targ, m_cpu, n, seed + s, variant=cfg["variant"], nthreads=threads,
                  surplus=False)
        if s >= warmup:
            times.append(time.perf_counter() - t0)
    value = m_cpu * n * len(times) / sum(times)
    return {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{m_cpu} chains x {n} samples per step, {cfg['variant']} executor, "
                      f"oracle/fsm_oracle.c with {threads} threads, surplus ticks skipped "
                      f"(as the device runs)"}, times


def run_reference_arm(args, cfg, rank):
    if rank != 0:
        return
    cb, times = cpu_baseline(cfg, steps=args.steps, warmup=args.warmup)
    v = cb["value"]
    line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "m": cfg["m_cpu"], "n": cfg["n"],
                       "d": cfg["d"]},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", "--chains", dest="m", type=int, default=0, help="override chains per GPU")
    ap.add_argument("--n", "--samples", dest="n", type=int, default=0,
                    help="override samples per chain")
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--no-lockstep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end legs (A/B runs)")
    ap.add_argument("--one-device", action="store_true",
                    help="tests: run every torchrun rank on cuda:0 with gloo collectives")
    ap.add_argument("--draw-window", type=int, default=-1,
                    help="DRMH pre-drawn window in draws (0: inline generator; -1: config default)")
    ap.add_argument("--draw-parts", type=int, default=-1,
                    help="DRMH windows: 1..8 chain parts overlapped on their own streams, 0 = "
                         "pipelined windows (double-buffered draws), -1: config default")
    ap.add_argument("--prior-parts", type=int, default=0,
                    help="ESS batched prior: chain parts overlapped on their own streams (0: config)")
    ap.add_argument("--prior", default="", choices=["", "none", "dmma", "trmm", "gemm", "device"],
                    help="ESS dense prior: batched nu = L eps per round (default: config's)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.m:
        cfg["m"] = args.m
    if args.n:
        cfg["n"] = args.n
    if args.draw_window >= 0:
        cfg["draw_window"] = args.draw_window
    if not args.lanes and cfg.get("lanes"):
        args.lanes = cfg["lanes"]     # e.g. C1: 128 chains, a whole block per chain
    if args.draw_parts >= 0:
        cfg["draw_parts"] = args.draw_parts
    if args.prior_parts:
        cfg["prior_parts"] = args.prior_parts
    if args.prior:
        cfg["prior_transform"] = None if args.prior == "none" else args.prior
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2503_17405_b200 as fm
    from paper_2503_17405_b200 import analysis, distributed

    if args.one_device:
        # functional check of the multi-rank path on a one-GPU box: every rank
        # on cuda:0, gloo collectives on host tensors (ranks never wait on one
        # another inside a kernel); its timings say nothing about scaling
        local = 0
    torch.cuda.set_device(local)
    backend = "gloo" if args.one_device else "nccl"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    coll_dev = dev if backend == "nccl" else torch.device("cpu")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    bundle, target = make_workload(cfg, fm)
    m, n, d = cfg["m"], cfg["n"], cfg["d"]
    off = rank * m
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    evaluator = None
    if cfg.get("batched"):
        from paper_2503_17405_b200.dense import LogisticRegressionEvaluator
        evaluator = LogisticRegressionEvaluator(*logreg_data(cfg), precision=cfg["batched"])

    def one_step(seed, timing=None):
        batch = fm.init_batch(bundle, target, m, seed, chain_offset=off)
        return fm.run_fsm_batched(bundle, target, batch, n, step_variant=cfg["variant"],
                                  output="torch", surplus=False, lanes=args.lanes,
                                  evaluator=evaluator, draw_window=cfg.get("draw_window", 0),
                                  prior_transform=cfg.get("prior_transform"),
                                  draw_parts=cfg.get("draw_parts", 1),
                                  prior_parts=cfg.get("prior_parts", 1),
                                  precision=cfg.get("precision", "fp64"),
                                  stop_sync=distributed.stop_sync() if world > 1 else None,
                                  _timing=timing)

    held = None
    for s in range(args.warmup):
        # keep the previous step's outputs alive exactly as the timed loop
        # does, so the allocator holds both sample buffers before timing
        held = one_step(1000 + s)
    barrier()
    from paper_2503_17405_b200 import _lib
    launches0 = _lib.lib().fsmc_launch_count()
    clocks = ClockSampler(local)
    step_ms, kern_ms = [], []
    samples = ledger = None
    for s in range(args.steps):
        flush.fill_(s & 0xff)          # evict L2 between timed steps (outside the window)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        timing = {}
        e0.record()
        samples, ledger = one_step(s, timing)
        e1.record()
        barrier()
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(timing["run_kernel_ms"])
        held = None
    clk = clocks.stop()
    launches = _lib.lib().fsmc_launch_count() - launches0    # libfsmc kernels in the timed steps
    t_total = max_over_ranks(sum(step_ms) / 1e3)
    value = world * m * n * args.steps / t_total
    ms_per_step = 1e3 * t_total / args.steps

    # ESS / R-hat of the last step's samples: per-rank partials, all-reduced
    burn = n // 10
    has_ess = n - burn >= 10
    ess_pooled = ess_per_sec = rhat_max = None
    if has_ess:
        mom = analysis.diag_moments(samples, burn=burn)
        if world > 1:
            loc = distributed.LocalMoments(mom.n, analysis_chain_means(samples, burn),
                                           mom.max_chain_var, mom.acov_tile, mom.acov_all)
            mom = distributed.allreduce_moments(loc, device=coll_dev)
        ess = analysis.ess_from_moments(mom)
        ess_pooled = ess.pooled
        rhat_max = float(np.nanmax(analysis.rhat_from_moments(mom)))
        ess_per_sec = ess.pooled / (t_total / args.steps)

    # lock-step (vmap-style) baseline, same code, same chains
    # (batched configs: the same evaluator in fsmc_advance_lockstep rounds, a
    # barrier at every sample; n_lock samples per chain bound its run time)
    lock = None
    if not args.no_lockstep:
        lock_ms, lock_extra = [], {}
        n_lock = min(n, cfg.get("n_lock", n))
        for s in range(1 if cfg.get("batched") else 2):
            flush.fill_(s)
            barrier()
            batch = fm.init_batch(bundle, target, m, s, chain_offset=off)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, lled = fm.run_standard_batched(bundle, target, batch, n_lock, output="torch",
                                              lanes=args.lanes, evaluator=evaluator)
            e1.record()
            barrier()
            lock_ms.append(e0.elapsed_time(e1))
            lock_extra = dict(lled.extras)
        t_lock = max_over_ranks(min(lock_ms) / 1e3)
        lock_value = world * m * n_lock / t_lock
        lock = {"value": lock_value, "unit": "samples/s", "ms_per_step": 1e3 * t_lock,
                "speedup": value / lock_value, "n": n_lock, **lock_extra}
        lock.update(lockstep_accounting(args, cfg, fm, bundle, target, m, n_lock, off, ledger,
                                        t_lock, value, lock_value, barrier, max_over_ranks, world,
                                        evaluator))

    # end-to-end through the public API as a drop-in caller gets it: the start
    # point from (pinned) host memory, init_batch, run_fsm_batched with the
    # reference's output types -- samples [n, m, d] float64 and the ledger's
    # int64 count matrices as host numpy arrays (output="numpy")
    x0_host = torch.zeros(d, dtype=torch.float64).pin_memory()

    def e2e_run(s, output):
        x0 = x0_host.to(dev, non_blocking=True)
        batch = fm.init_batch(bundle, target, m, 500 + s, x0=x0, chain_offset=off)
        return fm.run_fsm_batched(bundle, target, batch, n, step_variant=cfg["variant"],
                                  output=output, surplus=False, lanes=args.lanes,
                                  evaluator=evaluator, draw_window=cfg.get("draw_window", 0),
                                  prior_transform=cfg.get("prior_transform"),
                                  draw_parts=cfg.get("draw_parts", 1),
                                  prior_parts=cfg.get("prior_parts", 1),
                                  precision=cfg.get("precision", "fp64"))

    # e2e legs: >= 3 untimed warm-up calls (the first also pins the host buffers), then the
    # mean over up to 5 timed calls (1 warm-up + 2 timed when a device step exceeds 5 s: C5)
    long_step = ms_per_step > 5000.0
    e2e_warm = 1 if long_step else max(3, min(args.warmup, 5))
    e2e_timed = 2 if long_step else max(2, min(args.steps, 5))
    e2e_s, led_h = [], None
    for s in range(0 if args.no_e2e else e2e_warm + e2e_timed):
        smp = led_h = None
        barrier()
        t0 = time.perf_counter()
        smp, led_h = e2e_run(s, "numpy")
        barrier()
        e2e_s.append(time.perf_counter() - t0)
    if args.no_e2e:
        e2e_s = [float("nan")] * 2
        smp = np.zeros(0)
        led_h = type("L", (), {"loop_exec_counts": {}, "iter_counts": np.zeros(0),
                               "block_exec_counts": np.zeros(0)})()
    if not args.no_e2e:
        e2e_s = e2e_s[e2e_warm:]
    t_e2e = max_over_ranks(statistics.mean(e2e_s))
    d2h = smp.nbytes + sum(a.nbytes for a in led_h.loop_exec_counts.values()) + \
        led_h.iter_counts.nbytes + np.asarray(led_h.block_exec_counts).nbytes + 8 * (7 * m + 1)
    e2e = {"value": world * m * n / t_e2e, "unit": "samples/s", "h2d_bytes_per_step": 8 * d,
           "d2h_bytes_per_step": int(d2h),
           "includes": "init_batch (host start point) + run_fsm_batched(output='numpy'): samples "
                       "[n, m, d] f64 and the ledger's int64 count matrices delivered to host "
                       "memory (sample rows streamed out during the run where the windowed "
                       "DRMH path allows)",
           "warmup": 0 if args.no_e2e else e2e_warm, "steps": len(e2e_s), "stat": "mean",
           "ms": [round(1e3 * v, 3) for v in e2e_s]}
    del smp, led_h
    # the same with the samples left in HBM (output="torch"), plus the device ESS
    e2e_dev = [float("nan")] if args.no_e2e else []
    for s in range(0 if args.no_e2e else e2e_warm + e2e_timed):
        barrier()
        t0 = time.perf_counter()
        smp, _ = e2e_run(10 + s, "torch")
        if has_ess:
            _ = fm.effective_sample_size(smp, burn=burn).pooled
        else:
            _ = smp.mean(dim=(0, 1)).cpu()
        del smp
        barrier()
        e2e_dev.append(time.perf_counter() - t0)
    if not args.no_e2e:
        e2e_dev = e2e_dev[e2e_warm:]
    t_dev = max_over_ranks(statistics.mean(e2e_dev))
    e2e_device = {"value": world * m * n / t_dev, "unit": "samples/s",
                  "includes": "init_batch + run_fsm_batched(output='torch') + "
                              "effective_sample_size on the device; samples stay in HBM"}

    # roofline of the run (fsm_run_kernel, or drmh_draws_kernel + fsm_window_kernel
    # when the draws are generated ahead): algorithmic HBM bytes per launch
    kms = statistics.mean(kern_ms)
    evals = ledger.extras.get("evaluations", 0)
    proposals = int(ledger.iter_counts.sum().item()) if hasattr(ledger.iter_counts, "sum") else 0
    win = cfg.get("draw_window", 0) if cfg["family"] == "drmh" else 0
    st_bytes = 2 * m * 8 * (ledger_state_words(bundle, d))
    out_bytes = n * m * d * 8 + n * m * 4 * len(bundle.loop_states)
    draw_bytes = 2 * 8 * (d + 1) * proposals if win else 0     # written once, read once
    traffic_bytes = st_bytes + out_bytes + draw_bytes
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    pipe = json.load(open(os.path.join(ROOT, "profiles", "r01_pipe_peaks.json")))
    design = {"achieved": traffic_bytes / (kms / 1e3) / 1e9, "unit": "GB/s",
              "frac": traffic_bytes / (kms / 1e3) / 1e9 / peaks["hbm_gbs"],
              "algorithmic_bytes": traffic_bytes,
              "note": ("bytes this design moves: samples, ledger rows, chain state once per "
                       "launch and (windowed) the pre-drawn normals/uniforms at 16 B per draw "
                       "(written by drmh_draws_kernel, read by fsm_window_kernel)") if win else
                      ("bytes this design moves: samples, ledger rows and chain state loaded/"
                       "stored once per launch; the per-chain FSM state stays in registers or "
                       "shared memory for the whole run")}
    if draw_bytes:
        design["frac_without_draws"] = (st_bytes + out_bytes) / (kms / 1e3) / 1e9 / peaks["hbm_gbs"]
    # roofline.achieved follows SURVEY.md 8(d): its per-unit bytes (the traffic an
    # SoA-state-in-HBM step kernel moves per chain-tick, or per INTEGRATE
    # chain-tick for NUTS) x the units this run executed / the kernels' time.
    # This engine keeps that state on chip, so it is the bandwidth-equivalent
    # rate of the state-model, not DRAM traffic (that is `traffic`).
    n_inner = int(ledger.iter_counts.sum().item()) if hasattr(ledger.iter_counts, "sum") else 0
    fp = 4 if cfg.get("precision") == "fp32" else 8     # 8(d): bytes per float, parity / throughput
    if cfg["family"] == "ess":
        units, per_unit, uname = n_inner + 2 * n * m, 2 * d * fp + 96 + 3 * d * fp * n * m / \
            max(1, n_inner + 2 * n * m), "chain-tick (INIT, SHRINK, DONE)"
    elif cfg["family"] == "nuts":
        units, per_unit, uname = n_inner, 9.3 * d * fp + 100, "INTEGRATE chain-tick (leapfrog)"
    else:
        units, per_unit, uname = n_inner, 2 * d * fp + 96 + 2 * d * fp * n * m / max(1, n_inner), \
            "PROPOSE chain-tick"
    sm_ach = units * per_unit / (kms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": sm_ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": sm_ach / peaks["hbm_gbs"], "traffic": None,
            "kernel": ("drmh_draws_ilp_kernel<4> + fsm_window_kernel<DrmhWX,1,10,MOG,1>" if win else
                       "fsm_advance_kernel<Ess> rounds + prior_trmm_kernel (DMMA nu = L eps), every "
                       "launch of the run" if cfg.get("prior_transform") else
                       "fsm_run_kernel<%s>" % {"drmh": "Drmh", "ess": "Ess", "nuts": "Nuts"}.get(
                           cfg["family"], cfg["family"])),
            "kernel_ms": kms, "unit_of_work": uname, "units": units, "bytes_per_unit": per_unit,
            "algorithmic_bytes": units * per_unit,
            "source": "SURVEY.md 8(d) per-unit bytes x units / kernel time (CUDA events on the "
                      "launching stream)",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs", "design_traffic": design}
    if draw_bytes:
        tp = os.path.join(ROOT, "profiles", "r06_c2_traffic.json")      # every launch at HEAD
        if not os.path.exists(tp):
            tp = os.path.join(ROOT, "profiles", "r02_c2_traffic.json")
        if os.path.exists(tp) and cfg.get("draw_window") in (3300, 4070):
            # ncu DRAM bytes of the generator + window launches over a whole run, as a
            # multiple of their draw bytes (0.95 at HEAD: some draws still in L2), scaled
            # to this run by its draw bytes
            t = json.load(open(tp))
            roof["traffic"] = draw_bytes * t["measured_over_draw_bytes"]
            roof["traffic_source"] = os.path.relpath(tp, ROOT) + " (per launch pair: %.0f MB measured, "\
                "%.0f MB of draws)" % (t["measured_per_launch_pair"] / 1e6,
                                      t["algorithmic_draw_bytes_per_launch_pair"] / 1e6)
    tp3 = os.path.join(ROOT, "profiles", "r06_c3_traffic.json")     # every launch at HEAD
    if not os.path.exists(tp3):
        tp3 = os.path.join(ROOT, "profiles", "r03_c3_traffic.json")
    if cfg["family"] == "nuts" and not cfg.get("batched") and d == 100 and os.path.exists(tp3):
        # ncu DRAM bytes per chain-sample of the C3 run kernel, scaled to this run
        t = json.load(open(tp3))
        roof["traffic"] = t["measured_bytes_per_chain_sample"] * n * m
        roof["traffic_source"] = os.path.relpath(tp3, ROOT) + " (%.0f B per chain-sample measured)" \
            % t["measured_bytes_per_chain_sample"]
    tpc = os.path.join(ROOT, "profiles", "r06_%s_traffic.json" % args.config)
    if roof["traffic"] is None and not cfg.get("batched") and os.path.exists(tpc):
        # ncu DRAM bytes of every launch of the run's kernels per chain-sample, scaled
        t = json.load(open(tpc))
        roof["traffic"] = t["measured_bytes_per_chain_sample"] * n * m
        roof["traffic_source"] = os.path.relpath(tpc, ROOT) + " (%.0f B per chain-sample measured)" \
            % t["measured_bytes_per_chain_sample"]
    if cfg["family"] == "drmh" and proposals:
        # executed fp64 flops per DRMH proposal (DFMA = 2), from ncu SASS counts of
        # this pair of kernels (profiles/r05_c2_issue.json when present); peak =
        # measured DFMA rate
        ip = os.path.join(ROOT, "profiles", ISSUE_PROFILE)
        fpp, fsrc = FP64_FLOPS_PER_PROPOSAL, "profiles/r01b_c2_ncu.md"
        if win and cfg.get("precision") != "fp32" and os.path.exists(ip):
            t = json.load(open(ip))
            if t.get("fp64_flops_per_proposal"):
                fpp, fsrc = t["fp64_flops_per_proposal"], "profiles/" + ISSUE_PROFILE
        fl = fpp * proposals
        ach_tf = fl / (kms / 1e3) / 1e12
        roof["compute"] = {"pipe": "fp64", "achieved": ach_tf, "peak": pipe["fp64_fma_tflops"],
                           "unit": "TFLOP/s", "frac": ach_tf / pipe["fp64_fma_tflops"],
                           "flops_per_proposal": fpp, "flops_source": fsrc, "proposals": proposals,
                           "peak_source": "profiles/r01_pipe_peaks.json (tools/peak_probe.cu)"}
        if win and cfg.get("precision") != "fp32" and os.path.exists(ip):
            # warp instructions per proposal of the two kernels (ncu sm__inst_executed
            # over a profiled run / that run's proposals) against the issue ceiling:
            # 148 SMs x 4 schedulers x one warp instruction per cycle at this run's clock
            t = json.load(open(ip))
            mhz = clk.get("sm_mhz") or pipe.get("sm_mhz", 1965.0)
            slots = 148 * 4 * mhz * 1e6 * (kms / 1e3)
            ins = t["warp_inst_per_proposal"] * proposals
            roof["issue"] = {"warp_inst_per_proposal": t["warp_inst_per_proposal"],
                             "achieved": ins / slots, "frac": ins / slots,
                             "unit": "fraction of issue slots (148 SM x 4 schedulers x clock)",
                             "sm_mhz": mhz, "source": "profiles/" + ISSUE_PROFILE}

    if cfg.get("batched"):
        # dominant work: the two contractions per evaluation, 4 N d flops each
        flops = 4.0 * cfg["n_obs"] * d * evals
        ach = flops / (kms / 1e3) / 1e12
        bf16 = cfg["batched"] in ("bf16-tc", "fp16-tc")      # same dense rate for fp16
        pk = peaks.get("bf16_tflops_sustained", 1395.2) * (1.0 if bf16 else 0.5)
        roof = {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                "frac": ach / pk, "traffic": None,
                "kernel": ("logreg_tc_kernel (fused tcgen05: S=Theta X^T, G+=R X in TMEM)"
                           if bf16 else "cuBLAS TF32 GEMMs + fsmc_logreg_epilogue") +
                          " + fsm_advance_kernel<Nuts,128,2>",
                "kernel_ms": kms, "algorithmic_flops": flops,
                "note": "peak = measured sustained dense bf16 (fp16 has the same dense rate; half of "
                        "it for TF32); whole run "
                        "(advance rounds + evaluations) timed"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, _ = cpu_baseline(cfg, steps=1, warmup=0)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": ("f32 (fp64 draws)" if cfg.get("precision") == "fp32" else
                          EVAL_DTYPE.get(cfg.get("batched"), "f64")), "data": "synthetic",
                "config": {"workload": cfg["workload"], "chains_per_gpu": m, "chains_total": m * world,
                           "n": n, "d": d, "variant": cfg["variant"],
                           "parallelism": f"chains sharded over {world} GPU(s), no data-path "
                                          "collective", "l2": "flushed between steps (256 MiB write)",
                           "surplus_ticks": "skipped (discarded by the reference)"},
                "ess_per_sec": ess_per_sec, "ess_pooled": ess_pooled, "rhat_max": rhat_max,
                "lockstep": lock, "e2e": e2e, "e2e_device": e2e_device, "roofline": roof,
                "cpu_baseline": cpu,
                "clocks": clk, "gpu_launches": launches,
                "tick_count": ledger.tick_count,
                "evaluations_per_step": evals, "rounds_per_step": ledger.extras.get("rounds"),
                "step_ms": [round(v, 3) for v in step_ms], "kernel_ms": [round(v, 3) for v in kern_ms]}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def lockstep_accounting(args, cfg, fm, bundle, target, m, n_lock, off, ledger, t_lock, value,
                        lock_value, barrier, max_over_ranks, world, evaluator):
    """What the lock-step speed-up is made of.

    R_of_m: the paper's efficiency bound E[max_j N_ij] / E[N_ij] (PAPER.md
    section 5; analysis.py:150-185) from this run's own per-sample loop
    counts: the speed-up a lock-step with the same per-iteration cost as the
    FSM would allow.  same_generator: the FSM with the lock-step kernel's
    draw source (inline generator, per-chain prior transform), so the two
    differ only in synchronisation.  barrier_us: one grid-wide barrier of the
    lock-step's cooperative grid, measured alone (fsmc_lockstep_barrier_probe);
    barriers_per_step counts the while-loop tests of single-loop machines,
    sum_i (max_j N_ij + 1)."""
    import torch
    from paper_2503_17405_b200 import lockstep as LS
    out = {}
    its = ledger.iter_counts[:n_lock].to(torch.float64)
    mx = its.max(dim=1).values
    r_of_m = float(mx.mean() / its.mean())
    out["R_of_m"] = r_of_m
    out["speedup_over_R"] = value / lock_value / r_of_m
    if evaluator is None:
        same = {}
        if cfg.get("draw_window"):
            same = {"draw_window": 0, "draw_parts": 1}
        elif cfg.get("prior_transform"):
            same = {"prior_transform": None}
        if same:
            ts = []
            for s in range(2):
                barrier()
                batch = fm.init_batch(bundle, target, m, 40 + s, chain_offset=off)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fm.run_fsm_batched(bundle, target, batch, n_lock, step_variant=cfg["variant"],
                                   output="torch", surplus=False, lanes=args.lanes,
                                   **{"draw_window": 0, "prior_transform": None, **same})
                e1.record()
                barrier()
                ts.append(e0.elapsed_time(e1) / 1e3)
            t_same = max_over_ranks(min(ts))
            v_same = world * m * n_lock / t_same
            out["same_generator"] = {"value": v_same, "ms_per_step": 1e3 * t_same,
                                     "speedup": v_same / lock_value,
                                     "speedup_over_R": v_same / lock_value / r_of_m,
                                     "options": same}
        if cfg["family"] == "drmh":
            # R(m) = 1 exactly: max_tries = 1 makes every sample one proposal, so
            # the lock-step / FSM ratio there is the synchronisation overhead alone
            # (same generator, same chains); R(m) x this predicts the speed-up
            b1 = fm.drmh_kernel(1, bundle.proposal_scale)
            ts = {}
            for kind in ("fsm", "lockstep"):
                best = []
                for s in range(2):
                    barrier()
                    bt = fm.init_batch(b1, target, m, 70 + s, chain_offset=off)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    if kind == "fsm":
                        fm.run_fsm_batched(b1, target, bt, n_lock, step_variant=cfg["variant"],
                                           output="torch", surplus=False, lanes=args.lanes)
                    else:
                        fm.run_standard_batched(b1, target, bt, n_lock, output="torch",
                                                lanes=args.lanes)
                    e1.record()
                    barrier()
                    best.append(e0.elapsed_time(e1))
                ts[kind] = max_over_ranks(min(best) / 1e3)
            ov = ts["lockstep"] / ts["fsm"]
            out["sync_overhead_at_R1"] = {
                "kernel": "drmh_kernel(max_tries=1): one proposal per sample, R(m) = 1",
                "fsm_ms": 1e3 * ts["fsm"], "lockstep_ms": 1e3 * ts["lockstep"], "ratio": ov,
                "predicted_speedup_same_generator": r_of_m * ov}
        batch = fm.init_batch(bundle, target, m, 60, chain_offset=off)
        bus = LS.lockstep_barrier_us(bundle, target, batch, lanes=args.lanes)
        out["barrier_us"] = bus
        if cfg["family"] in ("drmh", "ess"):
            nbar = int((mx + 1).sum())
            out["barriers_per_step"] = nbar
            out["barrier_share"] = nbar * bus * 1e-6 / t_lock
    return out


def analysis_chain_means(samples, burn):
    return samples[burn:].mean(dim=0).cpu().numpy()


def ledger_state_words(bundle, d):
    from paper_2503_17405_b200 import _lib
    fam = bundle.family
    n_vec = {1: 2, 2: 3}.get(fam, 12)
    n_scal = {1: 3, 2: 6}.get(fam, 3)
    return n_vec * d + n_scal + _lib.FSMC_NINT


if __name__ == "__main__":
    main()
