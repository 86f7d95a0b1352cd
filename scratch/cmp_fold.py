import json, sys, os
sys.path.insert(0, "/root/repo")
import bench
from paper_2504_21411_b200 import profiler as PR
from paper_2504_21411_b200.planner import profiles as P
from paper_2504_21411_b200.planner.profiles import TrainingConfig
from paper_2504_21411_b200.planner.search import SearchConfig, optimize
from paper_2504_21411_b200.runtime.config import MODEL_PRESETS
for name, cp in [("llama2-7b", "profiles/b200_cluster.json"), ("gpt2-medium", "profiles/b200_cluster_gpt2m.json")]:
    cfg = MODEL_PRESETS[name]
    old = P.load_model_profile(f"profiles/b200_model_{name}.json")
    meta = json.load(open(f"profiles/b200_model_{name}.meta.json"))
    new = PR.calibrated_model_profile(cfg, meta["activation"])
    for n in (1, 2, 4, 8):
        c, _ = bench.cluster_profile(n, cp)
        gb = 8 * n if name == "llama2-7b" else 16 * n
        for tag, prof in (("old", old), ("new", new)):
            pl = optimize(prof, c, TrainingConfig(global_batch=gb), SearchConfig())
            ks = sorted({(s.tp, s.dp, s.zero_stage, s.sp, s.recompute) for s in pl.layer_strategies})
            print(name, n, tag, pl.pp, pl.microbatch, ks, round(pl.predicted_iteration_time, 4), round(max(pl.predicted_stage_peak_memory)/1e9, 1))
