"""Norm backward A/B (run once per GALV_NORM_UNFUSED / GALV_NORM_NT setting; the library
reads them once per process).  CUDA events over 50 calls; 8192 x 4096 bf16 (x, dy, dres,
dx = 268 MB per call > L2)."""
import json, os, sys, torch
from paper_2504_21411_b200 import kernels as K
res = {"env": {k: os.environ.get(k) for k in ("GALV_NORM_UNFUSED", "GALV_NORM_NT")}}
for rows, cols, layer in [(8192, 4096, False), (16384, 4096, False), (16384, 1024, True),
                          (16384, 2048, True), (8192, 5120, False)]:
    x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
    g = torch.randn(cols, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(cols, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn_like(x); dres = torch.randn_like(x); dx = torch.empty_like(x)
    dg = torch.zeros(cols, device="cuda"); db = torch.zeros(cols, device="cuda")
    if layer:
        _, mean, rstd = K.layernorm_fwd(x, g, b, 1e-5)
        fn = lambda: K.layernorm_bwd(x, g, mean, rstd, dy, dg, db, dres=dres, dx=dx)
    else:
        _, rstd = K.rmsnorm_fwd(x, g, 1e-5)
        fn = lambda: K.rmsnorm_bwd(x, g, rstd, dy, dg, dres=dres, dx=dx)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        fn()
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    alg = 4 * rows * cols * 2
    res[f"{'ln' if layer else 'rms'}_{rows}x{cols}"] = {"us": round(us, 1), "GBps": round(alg / us / 1e3)}
print(json.dumps(res))
