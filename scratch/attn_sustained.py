import os, sys, math, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_21411_b200 import kernels as K
B, S, H, D = 2, 4096, 32, 128
qkv = torch.randn(B * S, 3 * H * D, device='cuda').bfloat16()
mk = lambda t, j: t.as_strided((B, S, H, D), (S * 3 * H * D, 3 * H * D, D, 1), j * H * D)
q, k, v = mk(qkv, 0), mk(qkv, 1), mk(qkv, 2)
o = torch.empty(B, S, H, D, device='cuda', dtype=torch.bfloat16); lse = torch.empty(B, H, S, device='cuda')
dqkv = torch.empty_like(qkv); dq, dk, dv = mk(dqkv, 0), mk(dqkv, 1), mk(dqkv, 2)
do = torch.randn_like(o)
ws = torch.empty(K.attn_bwd_workspace_bytes(B, S, H, D, torch.bfloat16), dtype=torch.uint8, device="cuda")
fl = 4 * B * H * S * S * D / 2
f = lambda: K.attn_fwd(q, k, v, o, lse, scale=1 / math.sqrt(D), causal=True)
g = lambda: K.attn_bwd(q, k, v, o, do, lse, dq, dk, dv, scale=1 / math.sqrt(D), causal=True, workspace=ws)
t0 = time.time()
while time.time() - t0 < 4:
    f(); g(); torch.cuda.synchronize()
for name, fn, mult in (("fwd", f, 1), ("bwd", g, 2.5)):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(30): fn()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 30
    print(f"{os.environ.get('GALV_LIB','default')[-28:]} {name} {ms:.3f} ms {mult*fl/ms/1e9:.0f} TF", flush=True)
