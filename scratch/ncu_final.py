"""One launch each of the step's dominant kernels at the bench shapes (for ncu --set full)."""
import os, sys, math, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_21411_b200 import kernels as K
T, h, F = 8192, 4096, 11008
x = torch.randn(T, h, device="cuda").bfloat16() * 0.5
w = (torch.randn(2 * F, h, device="cuda") / 64).bfloat16()
gu, hh = K.gemm_swiglu_fwd(x, w)                      # 1: gate|up + SwiGLU (fused)
wq = (torch.randn(3 * h, h, device="cuda") / 64).bfloat16()
qkv = K.gemm(x, wq, trans_b=True)                     # 2: QKV fwd (plain bf16 epilogue)
B, S, H, D = 2, 4096, 32, 128
mk = lambda t, j: t.as_strided((B, S, H, D), (S * 3 * H * D, 3 * H * D, D, 1), j * H * D)
q, k, v = mk(qkv, 0), mk(qkv, 1), mk(qkv, 2)
o = torch.empty(B, S, H, D, device="cuda", dtype=torch.bfloat16); lse = torch.empty(B, H, S, device="cuda")
K.attn_fwd(q, k, v, o, lse, scale=1 / math.sqrt(D), causal=True)   # 3
dqkv = torch.empty_like(qkv); do = torch.randn_like(o)
K.attn_bwd(q, k, v, o, do, lse, mk(dqkv, 0), mk(dqkv, 1), mk(dqkv, 2), scale=1 / math.sqrt(D), causal=True)  # 4,5,6
torch.cuda.synchronize()
