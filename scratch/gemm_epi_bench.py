import sys, torch
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e)/it
for (M,N,Kd) in [(8192,12288,4096),(8192,4096,4096),(8192,22016,4096),(8192,4096,11008),(16384,4096,1024)]:
    a=torch.randn(M,Kd,device='cuda').bfloat16(); b=torch.randn(N,Kd,device='cuda').bfloat16()
    c=torch.empty(M,N,device='cuda',dtype=torch.bfloat16); c2=torch.empty_like(c)
    ptrs=torch.tensor([c2.data_ptr()],dtype=torch.int64,device='cuda')
    t1=bench(lambda: K.gemm(a,b,c,trans_b=True))
    t2=bench(lambda: K.gemm_rs(a,b,ptrs,M,0,trans_b=True,ldc=N))
    torch.cuda.synchronize()
    print(f"M{M} N{N} K{Kd}: direct-store epilogue {2*M*N*Kd/t1/1e9:.0f} TF | staged 256B-row epilogue {2*M*N*Kd/t2/1e9:.0f} TF | equal={torch.equal(c,c2)}", flush=True)
