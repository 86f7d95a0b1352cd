import sys, os, time, torch
sys.path.insert(0, '.')
from paper_2504_21411_b200.runtime.config import MODEL_PRESETS, uniform_config
from paper_2504_21411_b200.planner.strategy import ParallelStrategy
from paper_2504_21411_b200.planner.profiles import TrainingConfig
from paper_2504_21411_b200.runtime.engine import construct_hybrid_parallel_model
from paper_2504_21411_b200.runtime.init import synthetic_tokens
cfg = MODEL_PRESETS['gpt2-medium']
hc = uniform_config(cfg, ParallelStrategy(1,1,0,False,False), microbatch=16, n_microbatches=1)
m = construct_hybrid_parallel_model(cfg, hc, training=TrainingConfig(global_batch=16), init="fast")
tok = synthetic_tokens(cfg, 16).cuda()
for _ in range(3): m.train_step(tok)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): m.train_step(tok)
torch.cuda.synchronize()
print("wall ms/step", (time.perf_counter()-t0)/5*1e3)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    m.train_step(tok); torch.cuda.synchronize()
ka = prof.key_averages()
tot = sum(k.self_device_time_total for k in ka)
print("gpu busy ms", tot/1e3)
print(ka.table(sort_by="self_device_time_total", row_limit=18, max_name_column_width=50))
