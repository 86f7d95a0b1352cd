import sys, math, torch
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
def bench(fn, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e)/it
for (B,S,H,D) in [(2,4096,32,128),(1,32768,20,128),(16,1024,16,64)]:
    qkv = torch.randn(B*S, 3*H*D, device='cuda').bfloat16()
    mk = lambda j: qkv.as_strided((B,S,H,D),(S*3*H*D,3*H*D,D,1), j*H*D)
    q,k,v = mk(0),mk(1),mk(2)
    o = torch.empty(B,S,H,D,device='cuda',dtype=torch.bfloat16); lse=torch.empty(B,H,S,device='cuda')
    fl = 4*B*H*S*S*D/2
    ms = bench(lambda: K.attn_fwd(q,k,v,o,lse,scale=1/math.sqrt(D),causal=True))
    print(f"B{B} S{S} H{H} D{D} fwd {ms:.3f} ms {fl/ms/1e9:.0f} TF", flush=True)
