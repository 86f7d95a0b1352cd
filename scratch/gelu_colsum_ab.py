"""A/B: bias-GeLU bwd + colsum (two passes) vs the fused galv_bias_gelu_bwd_colsum, and the
norm backward fused vs two-kernel is covered by GALV_NORM_UNFUSED in bench.py.
CUDA events, 50 iterations after warm-up, inputs > L2 per iteration (rows x 4h bf16)."""
import json, torch
from paper_2504_21411_b200 import kernels as K

def timeit(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3  # us

out = []
for rows, cols in [(16384, 4096), (16384, 8192), (8192, 8192)]:
    x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn_like(x); dx = torch.empty_like(x)
    b = torch.randn(cols, device="cuda", dtype=torch.bfloat16)
    db = torch.zeros(cols, device="cuda")
    two = timeit(lambda: (K.bias_gelu_bwd(x, b, dy, dx), K.colsum(dx, db)))
    one = timeit(lambda: K.bias_gelu_bwd_colsum(x, b, dy, db, dx))
    bytes_ = 3 * rows * cols * 2
    r = {"shape": [rows, cols], "two_pass_us": two, "fused_us": one,
         "fused_GBps": bytes_ / one / 1e3, "algorithmic_bytes": bytes_}
    print(json.dumps(r)); out.append(r)
