"""Sustained GEMM sweep over one Llama-2-7B layer's GEMM shapes (mb2: 8192 tokens).
Run with GALV_GEMM_RASTER="group,gdim,hint" to compare raster / cache-hint variants.
Prints per-shape TF/s (after a ~2 s power-settling warm loop) and the layer aggregate."""
import os, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_21411_b200 import kernels as K

T = int(os.environ.get("TOK", 8192))
h, f = 4096, 11008
shapes = [  # name, M, N, K, trans_a, trans_b
    ("qkv_fwd", T, 3 * h, h, False, True), ("o_fwd", T, h, h, False, True),
    ("gu_fwd", T, 2 * f, h, False, True), ("down_fwd", T, h, f, False, True),
    ("qkv_dgrad", T, h, 3 * h, False, False), ("o_dgrad", T, h, h, False, False),
    ("gu_dgrad", T, h, 2 * f, False, False), ("down_dgrad", T, f, h, False, False),
    ("qkv_wgrad", 3 * h, h, T, True, False), ("o_wgrad", h, h, T, True, False),
    ("gu_wgrad", 2 * f, h, T, True, False), ("down_wgrad", h, f, T, True, False),
]
only = os.environ.get("ONLY")
bufs = []
for name, M, N, Kd, ta, tb in shapes:
    if only and name not in only.split(","):
        continue
    a = torch.randn(*((Kd, M) if ta else (M, Kd)), device="cuda").bfloat16()
    b = torch.randn(*((N, Kd) if tb else (Kd, N)), device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    bufs.append((name, M, N, Kd, ta, tb, a, b, c))

IMPL = os.environ.get("IMPL", "galv")
def run(x):
    name, M, N, Kd, ta, tb, a, b, c = x
    if IMPL == "cublas":
        torch.matmul(a.t() if ta else a, b.t() if tb else b, out=c)
    else:
        K.gemm(a, b, c, trans_a=ta, trans_b=tb)

# power-settling warm loop
t0 = time.time()
while time.time() - t0 < float(os.environ.get("WARM", 3)):
    for x in bufs:
        run(x)
    torch.cuda.synchronize()
res = {}
tot_f = tot_ms = 0.0
reps = int(os.environ.get("REPS", 8))
for rnd in range(2):
    for x in bufs:
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            run(x)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        fl = 2.0 * x[1] * x[2] * x[3]
        if rnd == 1:
            res[x[0]] = round(fl / ms / 1e9, 1)
            tot_f += fl; tot_ms += ms
print(json.dumps({"impl": IMPL, "variant": os.environ.get("GALV_GEMM_RASTER", "default"),
                  "layer_tflops": round(tot_f / tot_ms / 1e9, 1), **res}), flush=True)
