"""Kernel-level A/B: attention backward with the inverse RoPE in the dq/dk epilogues vs the
plain backward + the standalone inverse RoPE over dq|dk (Llama-2-7B shapes, mb 2)."""
import json, math, torch
from paper_2504_21411_b200 import kernels as K
B, S, H, D = 2, 4096, 32, 128
torch.manual_seed(0)
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
q, k, v = (qkv.view(B, S, 3, H, D)[:, :, i] for i in range(3))
o = torch.empty(B, S, H, D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B, H, S, device="cuda")
K.attn_fwd(q, k, v, o, lse, scale=1 / math.sqrt(D), causal=True)
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
dq, dk, dv = (dqkv.view(B, S, 3, H, D)[:, :, i] for i in range(3))
ws = torch.empty(K.attn_bwd_workspace_bytes(B, S, H, D, qkv.dtype), dtype=torch.uint8, device="cuda")
def fused():
    K.attn_bwd(q, k, v, o, do, lse, dq, dk, dv, scale=1 / math.sqrt(D), workspace=ws, rope_theta=1e4, rope_epilogue=True)
def default():
    K.attn_bwd(q, k, v, o, do, lse, dq, dk, dv, scale=1 / math.sqrt(D), workspace=ws, rope_theta=1e4)
def pair():
    K.attn_bwd(q, k, v, o, do, lse, dq, dk, dv, scale=1 / math.sqrt(D), workspace=ws)
def rope_only():
    K.rope_(dqkv.view(B * S, 3 * H, D)[:, :2 * H], S, theta=1e4, inverse=True)
def t(fn, n=40):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
res = {}
for rep in range(2):
    res[f"fused_us_{rep}"] = t(fused)
    res[f"bwd_only_us_{rep}"] = t(pair)
    res[f"rope_only_us_{rep}"] = t(rope_only)
    res[f"default_us_{rep}"] = t(default)
res["shape"] = [B, S, H, D]
print(json.dumps(res))
