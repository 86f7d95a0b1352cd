"""GEMM numerics vs a torch fp32 reference of the same op (GPU)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(a, b, ta, tb):
    A = a.float().t() if ta else a.float()
    B = b.float().t() if tb else b.float()
    return A @ B


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", [(128, 256, 64), (296, 520, 200), (1024, 768, 4096),
                                   (72, 1000, 136), (4096, 4096, 512)])
def test_gemm_bf16_tcgen05(ta, tb, shape):
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(0)
    M, N, Kd = shape
    a = torch.randn(*((Kd, M) if ta else (M, Kd)), device="cuda").bfloat16()
    b = torch.randn(*((N, Kd) if tb else (Kd, N)), device="cuda").bfloat16()
    ref = _ref(a, b, ta, tb)
    out = K.gemm(a, b, trans_a=ta, trans_b=tb, out_dtype=torch.float32)
    torch.cuda.synchronize()
    err = (out - ref).norm() / ref.norm()
    assert err < 1e-5, f"rel err {err}"  # fp32 accumulate of exact bf16 products
    outb = K.gemm(a, b, trans_a=ta, trans_b=tb)
    assert ((outb.float() - ref).norm() / ref.norm()) < 8e-3


def test_gemm_bf16_epilogue_bias_accumulate():
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(1)
    a = torch.randn(512, 384, device="cuda").bfloat16()
    w = torch.randn(640, 384, device="cuda").bfloat16()
    bias = torch.randn(640, device="cuda").bfloat16()
    c = torch.randn(512, 640, device="cuda")
    ref = c + 0.5 * (a.float() @ w.float().t()) + bias.float()
    K.gemm(a, w, c, trans_b=True, alpha=0.5, accumulate=True, bias=bias)
    assert ((c - ref).norm() / ref.norm()) < 1e-5


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_gemm_fp32_exact(ta, tb):
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(2)
    M, N, Kd = 130, 70, 300
    a = torch.randn(*((Kd, M) if ta else (M, Kd)), device="cuda", dtype=torch.float64)
    b = torch.randn(*((N, Kd) if tb else (Kd, N)), device="cuda", dtype=torch.float64)
    ref = _ref(a.double(), b.double(), ta, tb).double()
    A = a.t() if ta else a
    B = b.t() if tb else b
    ref = A @ B
    out = K.gemm(a.float(), b.float(), trans_a=ta, trans_b=tb)
    assert ((out.double() - ref).norm() / ref.norm()) < 1e-6
