"""Cost-model predictions (calibrated B200 profile) for every BASELINE config at 8 GPUs."""
import json, sys
sys.argv = ['x']; sys.path.insert(0, '.')
import bench
from paper_2504_21411_b200.runtime.config import MODEL_PRESETS
out = {}
cases = [("llama2-7b", 8, None, None), ("gpt2-medium", 16, None, None),
         ("gpt2-medium", 16, "dp8z3", 16), ("gpt-1.3b", 8, "tp8,dp8z3,tp4dp2", 8),
         ("llama2-13b", 1, None, None)]
for name, spg, pattern, mb in cases:
    cfg = MODEL_PRESETS[name]
    prof = ('profiles/b200_cluster_gpt2m.json' if name.startswith('gpt2') else
            'profiles/b200_cluster_llama13b.json' if name == 'llama2-13b' else
            'profiles/b200_cluster.json')
    c, _ = bench.cluster_profile(8, prof)
    gb = spg * 8
    if pattern:
        plan, hc, tr = bench.explicit_plan(cfg, 8, gb, c, pattern, mb)
    else:
        plan, hc, tr = bench.plan_for(cfg, 8, gb, c)
    t = plan.predicted_iteration_time
    tok = gb * cfg.seq_len / t
    key = f"{name}" + (f" [{pattern}]" if pattern else " [searched]")
    out[key] = {"n_gpus": 8, "global_batch": gb, "plan": bench.describe(hc),
                "predicted_iteration_time_s": t, "predicted_tokens_per_s": tok,
                "predicted_mfu": tok * cfg.train_flops_per_token() / (8 * 2.25e15),
                "predicted_stage_peak_memory_gb": [m / 1e9 for m in plan.predicted_stage_peak_memory],
                "note": "cost-model PREDICTION with the measured profile (8 GPUs not available via gpurun)"}
    print(key, out[key]["plan"], round(t, 3), round(tok), round(out[key]["predicted_mfu"], 3))
json.dump(out, open('profiles/r01/predicted_n8.json', 'w'), indent=1)
