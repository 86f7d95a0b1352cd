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


@pytest.mark.parametrize("M,F,Kd", [(512, 1024, 256), (300, 200, 136), (100, 256, 64),
                                    (1024, 11008, 512), (640, 2752, 4096)])
def test_gemm_swiglu_fused(M, F, Kd):
    """SwiGLU fused into the gate|up GEMM epilogue (fwd) and the down-projection dgrad
    epilogue (bwd) vs the unfused GEMM + SwiGLU kernels (same bf16 roundings) and vs an
    fp32 torch reference.  M <= 128 exercises the unfused fallback inside the C ABI."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(0)
    x = torch.randn(M, Kd, device="cuda").bfloat16()
    w_gu = (torch.randn(2 * F, Kd, device="cuda") / Kd ** 0.5).bfloat16()
    w_dn = (torch.randn(Kd, F, device="cuda") / F ** 0.5).bfloat16()
    dy = torch.randn(M, Kd, device="cuda").bfloat16()
    gu, h = K.gemm_swiglu_fwd(x, w_gu)
    gu_ref = K.gemm(x, w_gu, trans_b=True)
    h_ref = K.swiglu_fwd(gu_ref)
    dgu = K.gemm_swiglu_bwd(dy, w_dn, gu_ref)
    dh_ref = K.gemm(dy, w_dn)
    dgu_ref = K.swiglu_bwd(gu_ref, dh_ref)
    torch.cuda.synchronize()
    assert torch.equal(gu, gu_ref)
    for got, want in ((h, h_ref), (dgu, dgu_ref)):  # MUFU sigmoid: bf16-ulp differences
        d = (got.float() - want.float()).abs()
        assert d.max().item() <= 1e-2 * want.float().abs().max().item() + 1e-6
        assert (d.norm() / want.float().norm()).item() < 4e-3
    # fp32 reference of the whole MLP activation path
    g32, u32 = (x.float() @ w_gu.float().t()).split(F, dim=1)
    h32 = torch.nn.functional.silu(g32) * u32
    assert ((h.float() - h32).norm() / h32.norm()).item() < 1e-2


@pytest.mark.parametrize("M,F,Kd", [(512, 4096, 1024), (300, 200, 136), (100, 256, 64)])
@pytest.mark.parametrize("bias_dt", [torch.bfloat16, torch.float32, None])
def test_gemm_bias_gelu_fused(M, F, Kd, bias_dt):
    """bias-GeLU fused into the fc1 GEMM epilogue and the fc2 dgrad epilogue vs the unfused
    GEMM + bias_gelu kernels and an fp32 torch reference (M <= 128: C-ABI fallback)."""
    from paper_2504_21411_b200 import kernels as K
    if bias_dt == torch.float32 and M <= 128:
        pytest.skip("the unfused fallback takes a bf16 bias")
    torch.manual_seed(0)
    x = torch.randn(M, Kd, device="cuda").bfloat16()
    w1 = (torch.randn(F, Kd, device="cuda") / Kd ** 0.5).bfloat16()
    w2 = (torch.randn(Kd, F, device="cuda") / F ** 0.5).bfloat16()
    b = None if bias_dt is None else (0.5 * torch.randn(F, device="cuda")).to(bias_dt)
    dy = torch.randn(M, Kd, device="cuda").bfloat16()
    pre, act = K.gemm_bias_gelu_fwd(x, w1, b)
    pre_ref = K.gemm(x, w1, trans_b=True)
    b16 = None if b is None else b.bfloat16()
    act_ref = K.bias_gelu_fwd(pre_ref, b16) if b is not None else K.bias_gelu_fwd(pre_ref, None)
    dpre = K.gemm_bias_gelu_bwd(dy, w2, pre_ref, b)
    dact_ref = K.gemm(dy, w2)
    dpre_ref = K.bias_gelu_bwd(pre_ref, b16, dact_ref)
    torch.cuda.synchronize()
    assert torch.equal(pre, pre_ref)
    for got, want in ((act, act_ref), (dpre, dpre_ref)):
        d = (got.float() - want.float()).abs()
        assert d.max().item() <= 2e-2 * want.float().abs().max().item() + 1e-6
        assert (d.norm() / want.float().norm()).item() < 6e-3
    bb = 0 if b is None else b.float()
    a32 = torch.nn.functional.gelu(x.float() @ w1.float().t() + bb, approximate="tanh")
    assert ((act.float() - a32).norm() / a32.norm()).item() < 1e-2


@pytest.mark.parametrize("shape", [(1024, 1024, 16384), (3072, 1024, 16384), (512, 768, 8192),
                                   (4096, 4096, 8192)])
@pytest.mark.parametrize("acc", [False, True])
def test_gemm_splitk(shape, acc):
    """Split-K path (narrow output, long K: the GPT-2-medium wgrads) vs fp32 torch, with the
    accumulate-into-bf16 semantics of the wgrad call; the heuristic's split count is checked
    to be > 1 for the small-output shapes."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(0)
    M, N, Kd = shape
    a = torch.randn(Kd, M, device="cuda").bfloat16()   # dY^T layout (trans_a)
    b = torch.randn(Kd, N, device="cuda").bfloat16()
    c0 = torch.randn(M, N, device="cuda").bfloat16()
    c = c0.clone()
    K.gemm(a, b, c, trans_a=True, accumulate=acc)
    ref = a.float().t() @ b.float() + (c0.float() if acc else 0)
    torch.cuda.synchronize()
    assert ((c.float() - ref).norm() / ref.norm()).item() < 8e-3
    if M * N <= 3072 * 1024:
        assert K._gemm_splits(M, N, Kd) > 1
    out32 = K.gemm(a, b, trans_a=True, out_dtype=torch.float32)
    assert ((out32 - a.float().t() @ b.float()).norm() / ref.norm()).item() < 1e-5


@pytest.mark.parametrize("M,heads,Kd,S", [(1024, 2, 512, 256), (300, 3, 256, 100),
                                          (128, 2, 128, 64), (4096, 4, 1024, 4096)])
def test_gemm_rope_qkv_fused(M, heads, Kd, S):
    """QKV GEMM with RoPE in the tcgen05 epilogue == the plain GEMM followed by the
    standalone RoPE kernel on the q|k heads (the same fp32 arithmetic on the stored bf16
    values; at most a 1-ulp bf16 difference where FMA contraction differs), and against a
    torch fp32 RoPE of the GEMM output.  M = 300 leaves a partial pair tile; M = 128 takes
    the unfused fallback; S = 100 is not a multiple of 8 (fallback too)."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(M + heads)
    D = 128
    x = (torch.randn(M, Kd, device="cuda") / Kd ** 0.5).to(torch.bfloat16)
    w = torch.randn(3 * heads * D, Kd, device="cuda").to(torch.bfloat16)
    got = K.gemm_rope_qkv(x, w, S, 2 * heads * D)
    ref = K.gemm(x, w, trans_b=True)
    K.rope_(ref[:, :2 * heads * D].unflatten(1, (2 * heads, D)), S)
    diff = (got.float() - ref.float()).abs()
    ulp = ref.float().abs().clamp_min(1e-30) * 2.0 ** -7
    assert bool((diff <= ulp).all()), diff.max().item()
    assert (got == ref).float().mean().item() > 0.99
    assert torch.equal(got[:, 2 * heads * D:], ref[:, 2 * heads * D:])  # v untouched
    # torch fp32 RoPE of the stored GEMM output
    plain = K.gemm(x, w, trans_b=True).float()
    qk = plain[:, :2 * heads * D].unflatten(1, (2 * heads, D))
    pos = (torch.arange(M, device="cuda") % S).float()
    inv = 1.0 / 10000.0 ** (torch.arange(0, D, 2, device="cuda").float() / D)
    ang = pos[:, None] * inv[None, :]
    c, s = ang.cos()[:, None, :], ang.sin()[:, None, :]
    a, b = qk[..., :D // 2], qk[..., D // 2:]
    want = torch.cat([a * c - b * s, b * c + a * s], -1).flatten(1)
    err = ((got[:, :2 * heads * D].float() - want).norm() / want.norm()).item()
    assert err < 1e-2


def test_splitk_workspace_query_matches_the_plan():
    """galv_gemm_splitk_workspace reports splits*M*N fp32 bytes exactly when the split-K
    planner splits (narrow-output long-K wgrad shapes), else 0."""
    from paper_2504_21411_b200 import kernels as K
    lib = K.load_library()
    for M, N, Kd in [(1024, 1024, 16384), (3072, 1024, 16384), (8192, 8192, 4096)]:
        s = K._gemm_splits(M, N, Kd)
        want = s * M * N * 4 if s > 1 else 0
        assert lib.galv_gemm_splitk_workspace(M, N, Kd) == want
    assert lib.galv_colsum_workspace(100, 64, 1) == 0
