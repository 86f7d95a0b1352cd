import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_21411_b200 import kernels as K
T, h, F = 8192, 4096, 11008
dy = torch.randn(T, h, device="cuda").bfloat16(); wd = torch.randn(h, F, device="cuda").bfloat16()
gu = torch.randn(T, 2 * F, device="cuda").bfloat16(); dgu = torch.empty_like(gu)
x = torch.randn(T, h, device="cuda").bfloat16(); w = torch.randn(2 * F, h, device="cuda").bfloat16()
hh = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
K.gemm_swiglu_bwd(dy, wd, gu, dgu)
K.gemm_swiglu_fwd(x, w, gu, hh)
torch.cuda.synchronize()
