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
T = 8192
# (name, N_out, K_in): wgrad dW[N_out, K_in] += dY[T, N_out]^T @ X[T, K_in]; dgrad dX[T,K_in] = dY[T,N_out] @ W[N_out,K_in]
for name, No, Ki in [("qkv", 12288, 4096), ("o", 4096, 4096), ("gate_up", 22016, 4096), ("down", 4096, 11008), ("lm_head", 32000, 4096)]:
    dy = torch.randn(T, No, device='cuda').bfloat16(); x = torch.randn(T, Ki, device='cuda').bfloat16()
    w = torch.randn(No, Ki, device='cuda').bfloat16()
    gw = torch.zeros(No, Ki, device='cuda').bfloat16(); dx = torch.empty(T, Ki, device='cuda').bfloat16()
    f = 2*T*No*Ki
    t1 = bench(lambda: K.gemm(dy, x, gw, trans_a=True, accumulate=True))
    t2 = bench(lambda: gw.addmm_(dy.t(), x))
    t3 = bench(lambda: K.gemm(dy, w, dx))
    t4 = bench(lambda: torch.matmul(dy, w, out=dx))
    t5 = bench(lambda: K.gemm(x, w, dy, trans_b=True))
    t6 = bench(lambda: torch.matmul(x, w.t(), out=dy))
    print(f"{name:8s} fwd galv {f/t5/1e9:5.0f} cublas {f/t6/1e9:5.0f} | dgrad galv {f/t3/1e9:5.0f} cublas {f/t4/1e9:5.0f} | wgrad(acc) galv {f/t1/1e9:5.0f} cublas {f/t2/1e9:5.0f} TF", flush=True)
