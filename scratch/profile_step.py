import sys, os, torch
sys.path.insert(0, '.')
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
from paper_2504_21411_b200.runtime.config import MODEL_PRESETS, uniform_config
from paper_2504_21411_b200.planner.strategy import ParallelStrategy
from paper_2504_21411_b200.planner.profiles import TrainingConfig
from paper_2504_21411_b200.runtime.engine import construct_hybrid_parallel_model
from paper_2504_21411_b200.runtime.init import synthetic_tokens
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = MODEL_PRESETS['llama2-7b'].with_(n_layers=L)
hc = uniform_config(cfg, ParallelStrategy(1,1,0,False,False), microbatch=2, n_microbatches=2)
m = construct_hybrid_parallel_model(cfg, hc, training=TrainingConfig(global_batch=4), init="fast")
tok = synthetic_tokens(cfg, 4).cuda()
print("loss0", m.train_step(tok).item())
for _ in range(2): m.train_step(tok)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.train_step(tok); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=60))
