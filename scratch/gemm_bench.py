import torch, sys
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
for (M,N,Kd) in [(8192,12288,4096),(8192,4096,4096),(8192,22016,4096),(8192,4096,11008)]:
    for ta,tb in [(False,True),(False,False),(True,False)]:
        a=torch.randn(*((Kd,M) if ta else (M,Kd)),device='cuda').bfloat16()
        b=torch.randn(*((N,Kd) if tb else (Kd,N)),device='cuda').bfloat16()
        c=torch.empty(M,N,device='cuda',dtype=torch.bfloat16)
        ms=bench(lambda: K.gemm(a,b,c,trans_a=ta,trans_b=tb))
        A=a.t() if ta else a; B=b.t() if tb else b
        ms2=bench(lambda: torch.matmul(A,B))
        print(f"M{M} N{N} K{Kd} ta{int(ta)} tb{int(tb)}: galv {ms:.3f} ms {2*M*N*Kd/ms/1e9:.0f} TF | cublas {ms2:.3f} ms {2*M*N*Kd/ms2/1e9:.0f} TF", flush=True)
