import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_21411_b200 import kernels as K
T, h, F = 8192, 4096, 11008
x = torch.randn(T, h, device="cuda").bfloat16(); w = torch.randn(2 * F, h, device="cuda").bfloat16()
wd = torch.randn(h, F, device="cuda").bfloat16(); dy = torch.randn(T, h, device="cuda").bfloat16()
gu = torch.empty(T, 2 * F, device="cuda", dtype=torch.bfloat16); hh = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
dgu = torch.empty_like(gu); dh = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
fns = {
    "fwd_fused": lambda: K.gemm_swiglu_fwd(x, w, gu, hh),
    "fwd_unfused": lambda: (K.gemm(x, w, gu, trans_b=True), K.swiglu_fwd(gu, hh)),
    "fwd_gemm_only": lambda: K.gemm(x, w, gu, trans_b=True),
    "bwd_fused": lambda: K.gemm_swiglu_bwd(dy, wd, gu, dgu),
    "bwd_unfused": lambda: (K.gemm(dy, wd, dh), K.swiglu_bwd(gu, dh, dgu)),
    "bwd_gemm_only": lambda: K.gemm(dy, wd, dh),
}
t0 = time.time()
while time.time() - t0 < 3:
    for f in fns.values(): f()
    torch.cuda.synchronize()
for rnd in range(2):
    for n, f in fns.items():
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): f()
        e.record(); torch.cuda.synchronize()
        if rnd: print(f"{n:14s} {s.elapsed_time(e)/10:.3f} ms", flush=True)
