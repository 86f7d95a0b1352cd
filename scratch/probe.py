import torch, time, os, subprocess
print(subprocess.run(["nvidia-smi"],capture_output=True,text=True).stdout)
print("cores", len(os.sched_getaffinity(0)))
dev="cuda"
def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e)/it
for (M,N,K) in [(8192,12288,4096),(8192,4096,4096),(8192,22016,4096),(8192,4096,11008),(4096,4096,8192),(16384,4096,4096)]:
    a=torch.randn(M,K,device=dev,dtype=torch.bfloat16); b=torch.randn(N,K,device=dev,dtype=torch.bfloat16)
    ms=bench(lambda: a@b.t())
    print("gemm",M,N,K, ms, 2*M*N*K/ms/1e9, "TFLOPs")
import torch.nn.functional as F
for B,H,S,D in [(1,32,4096,128),(2,32,4096,128),(8,16,1024,64)]:
    q=torch.randn(B,H,S,D,device=dev,dtype=torch.bfloat16,requires_grad=True)
    k=torch.randn_like(q,requires_grad=True); v=torch.randn_like(q,requires_grad=True)
    ms=bench(lambda: F.scaled_dot_product_attention(q,k,v,is_causal=True))
    fl=4*B*H*S*S*D/2
    print("sdpa fwd",B,H,S,D,ms, fl/ms/1e9)
    o=F.scaled_dot_product_attention(q,k,v,is_causal=True); g=torch.randn_like(o)
    ms=bench(lambda: torch.autograd.grad(F.scaled_dot_product_attention(q,k,v,is_causal=True),(q,k,v),g))
    print("sdpa fwd+bwd",ms, 3.5*fl/ms/1e9)
try:
    import flash_attn
    from flash_attn import flash_attn_func
    q=torch.randn(1,4096,32,128,device=dev,dtype=torch.bfloat16)
    ms=bench(lambda: flash_attn_func(q,q,q,causal=True))
    print("fa2", ms, 4*32*4096*4096*128/2/ms/1e9)
except Exception as ex: print("fa2 fail", ex)
