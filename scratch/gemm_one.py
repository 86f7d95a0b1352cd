import sys, torch
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
M, N, Kd = 8192, 22016, 4096   # Llama-2-7B gate|up forward at microbatch 2 x 4096 tokens
a = torch.randn(M, Kd, device='cuda').bfloat16()
b = torch.randn(N, Kd, device='cuda').bfloat16()
c = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
for _ in range(5):
    K.gemm(a, b, c, trans_b=True)
torch.cuda.synchronize()
ref = a[:256].float() @ b.float().t()
err = ((c[:256].float() - ref).norm() / ref.norm()).item()
print("rel err", err)
assert err < 1e-2
