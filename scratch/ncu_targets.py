"""Single launches of the dominant kernels for ncu --set full captures (profiles/r01)."""
import sys, math, torch
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
what = sys.argv[1]
if what == 'gemm':   # gate|up forward of Llama-2-7B at microbatch 2 x 4096: [8192,4096] x [22016,4096]^T
    a = torch.randn(8192, 4096, device='cuda').bfloat16()
    w = torch.randn(22016, 4096, device='cuda').bfloat16()
    for _ in range(3):
        c = K.gemm(a, w, trans_b=True)
    torch.cuda.synchronize()
elif what == 'attn':  # causal B2 S4096 H32 D128 fwd + bwd
    B, S, H, D = 2, 4096, 32, 128
    qkv = torch.randn(B*S, 3*H*D, device='cuda').bfloat16()
    mk = lambda j: qkv.as_strided((B,S,H,D),(S*3*H*D,3*H*D,D,1), j*H*D)
    q, k, v = mk(0), mk(1), mk(2)
    o = torch.empty(B,S,H,D,device='cuda',dtype=torch.bfloat16); lse=torch.empty(B,H,S,device='cuda')
    dqkv = torch.empty_like(qkv)
    dq, dk, dv = [dqkv.as_strided((B,S,H,D),(S*3*H*D,3*H*D,D,1), j*H*D) for j in range(3)]
    do = torch.randn_like(o)
    ws = torch.empty(K.attn_bwd_workspace_bytes(B,S,H,D,torch.bfloat16), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        K.attn_fwd(q,k,v,o,lse,scale=1/math.sqrt(D),causal=True)
        K.attn_bwd(q,k,v,o,do,lse,dq,dk,dv,scale=1/math.sqrt(D),causal=True,workspace=ws)
    torch.cuda.synchronize()
