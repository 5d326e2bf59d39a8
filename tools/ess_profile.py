import cProfile, pstats, sys, torch
sys.path.insert(0, ".")
import bench, paper_2503_17405_b200 as fm
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"])
bundle, target = bench.make_workload(cfg, fm)
batch = fm.init_batch(bundle, target, cfg["m"], 1)
smp, _ = fm.run_fsm_batched(bundle, target, batch, cfg["n"], step_variant=cfg["variant"], output="torch",
                            surplus=False, prior_transform=cfg.get("prior_transform"), lanes=cfg.get("lanes", 0))
torch.cuda.synchronize()
fm.effective_sample_size(smp, burn=cfg["n"] // 10); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
fm.effective_sample_size(smp, burn=cfg["n"] // 10); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
