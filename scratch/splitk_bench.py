import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_21411_b200 import kernels as K
shapes = [(1024, 1024, 16384), (3072, 1024, 16384), (4096, 1024, 16384), (1024, 4096, 16384),
          (4096, 4096, 8192), (12288, 4096, 8192), (4096, 11008, 8192), (2048, 2048, 16384)]
for M, N, Kd in shapes:
    a = torch.randn(Kd, M, device="cuda").bfloat16(); b = torch.randn(Kd, N, device="cuda").bfloat16()
    c = torch.zeros(M, N, device="cuda").bfloat16()
    sp = K._gemm_splits(M, N, Kd)
    def run(force1):
        if force1:
            K._SPLITS[(M, N, Kd)] = 1
        else:
            K._SPLITS[(M, N, Kd)] = sp
        K.gemm(a, b, c, trans_a=True, accumulate=True)
    res = []
    for force1 in (True, False):
        for _ in range(3): run(force1)
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20): run(force1)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 20
        res.append(f"{2*M*N*Kd/ms/1e9:.0f} TF")
    print(M, N, Kd, "splits", sp, "| no-split", res[0], "| split", res[1], flush=True)
