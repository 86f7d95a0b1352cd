import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_21411_b200 import kernels as K
for T, h in [(16384, 1024), (16384, 2048), (8192, 4096)]:
    F = 4 * h
    x = torch.randn(T, h, device="cuda").bfloat16(); w1 = (torch.randn(F, h, device="cuda") / h**.5).bfloat16()
    w2 = (torch.randn(h, F, device="cuda") / F**.5).bfloat16(); b = torch.randn(F, device="cuda").bfloat16()
    dy = torch.randn(T, h, device="cuda").bfloat16()
    pre = torch.empty(T, F, device="cuda", dtype=torch.bfloat16); act = torch.empty_like(pre); dpre = torch.empty_like(pre)
    cs = torch.zeros(F, device="cuda")
    fns = {
        "fwd_fused": lambda: K.gemm_bias_gelu_fwd(x, w1, b, pre, act),
        "fwd_unfused": lambda: (K.gemm(x, w1, pre, trans_b=True), K.bias_gelu_fwd(pre, b, act)),
        "bwd_fused": lambda: K.gemm_bias_gelu_bwd(dy, w2, pre, b, dpre),
        "bwd_unfused": lambda: (K.gemm(dy, w2, dpre), K.bias_gelu_bwd(pre, b, dpre, dpre)),
        "colsum": lambda: K.colsum(dpre, cs),
    }
    t0 = time.time()
    while time.time() - t0 < 1.5:
        for f in fns.values(): f()
        torch.cuda.synchronize()
    out = []
    for n, f in fns.items():
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): f()
        e.record(); torch.cuda.synchronize()
        out.append(f"{n} {s.elapsed_time(e)/10*1e3:.0f}us")
    print(T, h, " | ".join(out), flush=True)
