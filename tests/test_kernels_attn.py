"""Flash attention fwd/bwd vs a torch fp32 reference (GPU)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.double() - b.double()).norm() / (b.double().norm() + 1e-30)).item()


def ref_attn(q, k, v, causal):
    # q,k,v [B,S,H,D] fp32
    qt, kt, vt = (t.permute(0, 2, 1, 3) for t in (q, k, v))
    s = qt @ kt.transpose(-1, -2) / math.sqrt(q.shape[-1])
    if causal:
        S = q.shape[1]
        s = s.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1),
                          float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ vt
    return o.permute(0, 2, 1, 3), lse


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("S", [128, 200, 512])
@pytest.mark.parametrize("causal", [True, False])
def test_attention(dt, D, S, causal):
    if dt == torch.float32 and D != 64:
        pytest.skip("fp32 path is head_dim 64 (tiny config)")
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(0)
    B, H = 2, 3
    qkv = torch.randn(B, S, 3, H, D, device="cuda").to(dt)
    q, k, v = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]
    o = torch.empty(B, S, H, D, device="cuda", dtype=dt)
    lse = torch.empty(B, H, S, device="cuda")
    scale = 1 / math.sqrt(D)
    K.attn_fwd(q, k, v, o, lse, scale=scale, causal=causal)
    qr, kr, vr = (t.float().clone().requires_grad_(True) for t in (q, k, v))
    o_ref, lse_ref = ref_attn(qr, kr, vr, causal)
    tol = 1e-5 if dt == torch.float32 else 1e-2
    assert rel(o, o_ref) < tol
    assert rel(lse, lse_ref) < 1e-5 if dt == torch.float32 else 1e-3
    do = torch.randn_like(o_ref)
    o_ref.backward(do)
    dqkv = torch.empty_like(qkv)
    dq, dk, dv = dqkv[:, :, 0], dqkv[:, :, 1], dqkv[:, :, 2]
    K.attn_bwd(q, k, v, o, do.to(dt).contiguous(), lse, dq, dk, dv, scale=scale, causal=causal)
    for got, want in ((dq, qr.grad), (dk, kr.grad), (dv, vr.grad)):
        assert rel(got, want) < (1e-5 if dt == torch.float32 else 2e-2)


def test_attention_fwd_repeatable_rescale_heavy():
    """Regression: the softmax row-max exchange buffer once overlapped the O-done / V-empty
    mbarriers, which corrupted barrier state and intermittently faulted the forward.
    Sharply peaked, row-varying scores force lazy O rescales on most key blocks; the output
    must match the fp32 reference on every row (incl. rows 0-7 of each tile) and be
    bitwise repeatable across launches."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(1)
    B, S, H, D = 1, 1024, 4, 128
    qkv = torch.randn(B, S, 3, H, D, device="cuda")
    qkv[:, :, :2] *= torch.linspace(0.5, 6.0, S, device="cuda").view(1, S, 1, 1, 1)
    qkv = qkv.bfloat16()
    q, k, v = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]
    lse = torch.empty(B, H, S, device="cuda")
    scale = 1 / math.sqrt(D)
    o_ref, lse_ref = ref_attn(q.float(), k.float(), v.float(), True)
    first = None
    for _ in range(40):
        o = torch.empty(B, S, H, D, device="cuda", dtype=torch.bfloat16)
        K.attn_fwd(q, k, v, o, lse, scale=scale, causal=True)
        if first is None:
            first = o.clone()
            err_rows = ((o.float() - o_ref).norm(dim=-1) / (o_ref.norm(dim=-1) + 1e-6))
            assert err_rows.max().item() < 5e-2
            assert rel(lse, lse_ref) < 1e-3
        else:
            assert torch.equal(o, first)
    torch.cuda.synchronize()
