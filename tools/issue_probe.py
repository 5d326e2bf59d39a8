"""One C2 run (bench.py's configuration and run options, n samples per chain)
that prints its proposal count; under `ncu --metrics sm__inst_executed.sum,...`
it yields the warp instructions per DRMH proposal of the two hot kernels.

  ncu --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__cycles_active.avg,\
      sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,\
      sm__sass_thread_inst_executed_op_dfma_pred_on.sum \
      -k regex:"drmh_draws|fsm_window" --csv --log-file X.csv python tools/issue_probe.py 200 > P.json
  python tools/issue_probe.py --summarise X.csv P.json > profiles/r04_c2_issue.json
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(n):
    import torch
    import bench
    import paper_2503_17405_b200 as fm
    cfg = bench.CONFIGS["c2"]
    bundle, target = bench.make_workload(cfg, fm)
    batch = fm.init_batch(bundle, target, cfg["m"], 0)
    _, led = fm.run_fsm_batched(bundle, target, batch, n, step_variant=cfg["variant"],
                                output="torch", surplus=False, draw_window=cfg["draw_window"],
                                draw_parts=cfg["draw_parts"])
    torch.cuda.synchronize()
    print(json.dumps({"n": n, "m": cfg["m"], "proposals": int(led.iter_counts.sum().item()),
                      "draw_window": cfg["draw_window"], "draw_parts": cfg["draw_parts"]}))


def summarise(csv_path, probe_path):
    probe = json.loads(open(probe_path).read().strip().splitlines()[-1])
    rows = list(csv.DictReader(l for l in open(csv_path) if not l.startswith("==")))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    launches = collections.Counter()
    for r in rows:
        k = "drmh_draws_kernel" if "drmh_draws" in r["Kernel Name"] else "fsm_window_kernel"
        v = float(r["Metric Value"].replace(",", ""))
        agg[k][r["Metric Name"]] += v
        if r["Metric Name"] == "sm__inst_executed.sum":
            launches[k] += 1
    per = {k: agg[k]["sm__inst_executed.sum"] / probe["proposals"] for k in agg}
    dp = {}
    for k in agg:   # executed fp64 flops (DFMA counted twice) per proposal
        a = agg[k]
        dp[k] = (a.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0) +
                 a.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0) +
                 2 * a.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)) / probe["proposals"]
    out = {"what": "warp instructions executed per DRMH proposal (C2: MoG d=10, m=65536, "
                   f"windowed draws in {probe.get('draw_parts', 4)} parts), ncu sm__inst_executed.sum over "
                   "every launch of the profiled run / its proposals",
           "probe": probe, "launches": dict(launches),
           "warp_inst_per_proposal_by_kernel": per,
           "warp_inst_per_proposal": sum(per.values()),
           "fp64_flops_per_proposal_by_kernel": dp,
           "fp64_flops_per_proposal": sum(dp.values()),
           "totals": {k: dict(v) for k, v in agg.items()},
           "command": "tools/issue_probe.py (see its docstring)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--summarise":
        summarise(sys.argv[2], sys.argv[3])
    else:
        run(int(sys.argv[1]))
