"""Norm / RoPE / activation / embedding / cross-entropy / AdamW / reshard kernels vs
plain torch fp32 references of the same op (GPU)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu
DT = [torch.float32, torch.bfloat16]


def rel(a, b):
    return ((a.double() - b.double()).norm() / (b.double().norm() + 1e-30)).item()


def tol(dt):
    return 1e-5 if dt == torch.float32 else 1e-2


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("resid", [False, True])
def test_rmsnorm(dt, resid):
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(0)
    x = torch.randn(300, 1024, device="cuda").to(dt)
    r = torch.randn_like(x) if resid else None
    g = (1 + 0.1 * torch.randn(1024, device="cuda")).to(dt)
    ro = torch.empty_like(x) if resid else None
    y, rstd = K.rmsnorm_fwd(x, g, 1e-5, residual=r, res_out=ro)
    xs = (x.float() + r.float()) if resid else x.float()
    if resid:
        assert rel(ro, xs) < tol(dt)
        xs = ro.float()
    ref = xs * torch.rsqrt(xs.pow(2).mean(-1, keepdim=True) + 1e-5) * g.float()
    assert rel(y, ref) < tol(dt)
    # backward
    xr = xs.clone().requires_grad_(True)
    gr = g.float().clone().requires_grad_(True)
    out = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * gr
    dy = torch.randn_like(out)
    out.backward(dy)
    dg = torch.zeros(1024, device="cuda")
    src = ro if resid else x
    dres = torch.randn_like(x) if resid else None
    dx = K.rmsnorm_bwd(src, g, rstd, dy.to(dt), dg, dres=dres)
    want = xr.grad + (dres.float() if resid else 0)
    assert rel(dx, want) < tol(dt) * 2
    assert rel(dg, gr.grad) < tol(dt) * 2


@pytest.mark.parametrize("dt", DT)
def test_layernorm(dt):
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(1)
    x = (torch.randn(257, 512, device="cuda") * 2 + 0.5).to(dt)
    g = (1 + 0.1 * torch.randn(512, device="cuda")).to(dt)
    b = (0.1 * torch.randn(512, device="cuda")).to(dt)
    y, mean, rstd = K.layernorm_fwd(x, g, b, 1e-5)
    xr = x.float().clone().requires_grad_(True)
    gr = g.float().clone().requires_grad_(True)
    br = b.float().clone().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xr, (512,), gr, br, 1e-5)
    assert rel(y, ref) < tol(dt)
    dy = torch.randn_like(ref)
    ref.backward(dy)
    dg = torch.zeros(512, device="cuda")
    db = torch.zeros(512, device="cuda")
    dx = K.layernorm_bwd(x, g, mean, rstd, dy.to(dt), dg, db)
    assert rel(dx, xr.grad) < tol(dt) * 2
    assert rel(dg, gr.grad) < tol(dt) * 2
    assert rel(db, br.grad) < tol(dt) * 2


@pytest.mark.parametrize("layer", [False, True])
@pytest.mark.parametrize("rows,cols,off", [(3, 4096, 0), (2000, 4096, 1), (1500, 5120, 0),
                                           (700, 2048, 3), (5000, 1024, 0), (64, 8192, 2),
                                           # warp-per-row kernel (<= 1024 columns)
                                           (16384, 1024, 0), (999, 512, 1), (7, 768, 0),
                                           (100, 256, 2)])
def test_norm_bwd_fused_shapes(layer, rows, cols, off):
    """Fused dx+dgamma backward (persistent rows, smem partials, one atomic flush per CTA)
    across the model widths, rows not a multiple of the grid, and dgamma/dbeta views at
    offsets that are not 16-byte aligned (scalar-atomic flush)."""
    from paper_2504_21411_b200 import kernels as K
    if layer and cols > 4096:
        pytest.skip("LayerNorm widths > 4096 use the two-kernel path")
    torch.manual_seed(rows + cols)
    dt = torch.bfloat16
    x = (torch.randn(rows, cols, device="cuda") * 1.5 + 0.2).to(dt)
    g = (1 + 0.1 * torch.randn(cols, device="cuda")).to(dt)
    b = (0.1 * torch.randn(cols, device="cuda")).to(dt)
    dy = torch.randn(rows, cols, device="cuda").to(dt)
    dres = torch.randn(rows, cols, device="cuda").to(dt)
    xr = x.float().clone().requires_grad_(True)
    gr = g.float().clone().requires_grad_(True)
    br = b.float().clone().requires_grad_(True)
    if layer:
        y, mean, rstd = K.layernorm_fwd(x, g, b, 1e-5)
        ref = torch.nn.functional.layer_norm(xr, (cols,), gr, br, 1e-5)
    else:
        y, rstd = K.rmsnorm_fwd(x, g, 1e-5)
        ref = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * gr
    ref.backward(dy.float())
    buf = torch.zeros(2 * cols + 8, device="cuda")
    seed = torch.randn(cols, device="cuda")
    dg = buf[off:off + cols]
    dg.copy_(seed)  # accumulates into existing contents
    db = buf[off + cols + 4:off + 2 * cols + 4]
    if layer:
        dx = K.layernorm_bwd(x, g, mean, rstd, dy, dg, db, dres=dres)
        assert rel(db, br.grad) < 1e-4
    else:
        dx = K.rmsnorm_bwd(x, g, rstd, dy, dg, dres=dres)
    assert rel(dx, xr.grad + dres.float()) < 2e-2
    assert rel(dg - seed, gr.grad) < 1e-4


def rope_ref(x, S, theta=10000.0):
    T, H, D = x.shape
    pos = (torch.arange(T, device=x.device) % S).float()
    inv = 1.0 / theta ** (torch.arange(0, D, 2, device=x.device).float() / D)
    ang = pos[:, None] * inv[None, :]
    c, s = ang.cos()[:, None, :], ang.sin()[:, None, :]
    x1, x2 = x[..., : D // 2].float(), x[..., D // 2:].float()
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)


@pytest.mark.parametrize("dt", DT)
def test_rope_roundtrip(dt):
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(2)
    qkv = torch.randn(2 * 128, 3 * 4 * 64, device="cuda").to(dt)
    orig = qkv.clone()  # unaliased copy of the input
    view = qkv[:, : 4 * 64].view(256, 4, 64)
    ref = rope_ref(view.clone(), 128)
    K.rope_(view, 128)
    assert rel(view, ref) < tol(dt)
    # the rotated values are rounded to dt, so the round trip is exact only in fp32
    K.rope_(view, 128, inverse=True)
    assert rel(view, orig[:, : 4 * 64].view(256, 4, 64)) < (1e-6 if dt == torch.float32
                                                            else 1e-2)
    assert torch.equal(qkv[:, 4 * 64:], orig[:, 4 * 64:])  # v columns untouched


@pytest.mark.parametrize("dt", DT)
def test_swiglu_and_gelu(dt):
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(3)
    gu = torch.randn(100, 2 * 256, device="cuda").to(dt)
    h = K.swiglu_fwd(gu)
    g, u = gu.float()[:, :256].requires_grad_(True), gu.float()[:, 256:].requires_grad_(True)
    ref = torch.nn.functional.silu(g) * u
    assert rel(h, ref) < tol(dt)
    dh = torch.randn_like(ref)
    ref.backward(dh)
    dgu = K.swiglu_bwd(gu, dh.to(dt))
    assert rel(dgu[:, :256], g.grad) < tol(dt) * 2
    assert rel(dgu[:, 256:], u.grad) < tol(dt) * 2
    x = torch.randn(64, 128, device="cuda").to(dt)
    bias = torch.randn(128, device="cuda").to(dt)
    y = K.bias_gelu_fwd(x, bias)
    xr = x.float().clone().requires_grad_(True)
    r = torch.nn.functional.gelu(xr + bias.float(), approximate="tanh")
    assert rel(y, r) < tol(dt)
    dy = torch.randn_like(r)
    r.backward(dy)
    assert rel(K.bias_gelu_bwd(x, bias, dy.to(dt)), xr.grad) < tol(dt) * 2
    cs = torch.zeros(128, device="cuda")
    K.colsum(x, cs, accumulate=False)
    assert rel(cs, x.float().sum(0)) < 1e-5


@pytest.mark.parametrize("dt", DT)
def test_embedding_and_xent(dt):
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(4)
    V, Hd, T = 1000, 64, 300
    table = torch.randn(V, Hd, device="cuda").to(dt)
    ids = torch.randint(0, V, (T,), device="cuda")
    out = K.embed_fwd(ids, table)
    assert rel(out, table.float()[ids]) == 0
    dt_acc = torch.zeros(V, Hd, device="cuda")
    dout = torch.randn(T, Hd, device="cuda").to(dt)
    K.embed_bwd(ids, dout, dt_acc)
    ref = torch.zeros(V, Hd, device="cuda").index_add_(0, ids, dout.float())
    assert rel(dt_acc, ref) < 1e-6
    logits = (3 * torch.randn(T, V, device="cuda")).to(dt)
    labels = torch.randint(0, V, (T,), device="cuda")
    labels[5] = -100
    lr = logits.float().clone().requires_grad_(True)
    l_ref = torch.nn.functional.cross_entropy(lr, labels, reduction="none", ignore_index=-100)
    (l_ref.sum() / T).backward()
    stats = torch.empty(T, 3, device="cuda")
    loss = torch.empty(T, device="cuda")
    d = logits.clone()
    K.xent(d, labels, stats, 3, loss=loss, dlogits=d, grad_scale=1.0 / T)
    assert rel(loss, l_ref) < tol(dt)
    assert rel(d, lr.grad) < tol(dt) * 2


def test_adamw_matches_torch():
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(5)
    n = 10007
    p = torch.randn(n, device="cuda")
    grads = [torch.randn(n, device="cuda") for _ in range(3)]
    ref = p.clone().requires_grad_(True)
    opt = torch.optim.AdamW([ref], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
    master, m, v = p.clone(), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    out = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    for step, g in enumerate(grads, 1):
        ref.grad = g.clone()
        opt.step()
        K.adamw(master, m, v, g, out, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                weight_decay=0.1, step=step)
    assert rel(master, ref.detach()) < 1e-6
    assert rel(out, ref.detach()) < 1e-2


def test_gather_scatter_rows():
    from paper_2504_21411_b200 import kernels as K
    src = torch.randn(100, 64, device="cuda").bfloat16()
    idx = torch.randperm(100, device="cuda")[:37]
    dst = torch.empty(37, 64, device="cuda").bfloat16()
    K.gather_rows(src, idx, dst)
    assert torch.equal(dst, src[idx])
    back = torch.zeros_like(src)
    K.scatter_rows(dst, idx, back)
    assert torch.equal(back[idx], src[idx])


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("rows,cols", [(16384, 1024), (300, 4096), (7, 72), (1000, 130)])
def test_colsum_shapes(dt, rows, cols):
    """Column sums (bias gradients): vectorized path (16-byte rows) and the scalar fallback
    (cols*esize not a multiple of 16), accumulate semantics."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(5)
    x = torch.randn(rows, cols, device="cuda").to(dt)
    cs = torch.full((cols,), 0.5, device="cuda")
    K.colsum(x, cs, accumulate=True)
    want = x.double().sum(0) + 0.5
    assert ((cs.double() - want).norm() / want.norm()).item() < 1e-5


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("rows,cols", [(1000, 4096), (37, 1024), (4096, 8192), (5, 64)])
def test_bias_gelu_bwd_colsum(dt, rows, cols):
    """Fused bias-GeLU backward + bias gradient == galv_bias_gelu_bwd then galv_colsum
    (bitwise for dx; the column sums agree to fp32 reduction order), with the bias an
    unaligned view into a flat buffer as the runtime's parameter store hands it out."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(rows)
    x = torch.randn(rows, cols, device="cuda").to(dt)
    dy = torch.randn(rows, cols, device="cuda").to(dt)
    flat = torch.randn(cols + 3, device="cuda").to(dt)
    b = flat[3:]
    with pytest.raises(RuntimeError, match="aligned"):  # the vector kernel refuses it
        K.bias_gelu_bwd(x, b, dy)
    ref_dx = K.bias_gelu_bwd(x, b.clone(), dy)
    ref_db = torch.full((cols,), 0.25, device="cuda")
    K.colsum(ref_dx, ref_db, accumulate=True)
    db = torch.full((cols,), 0.25, device="cuda")
    dx = K.bias_gelu_bwd_colsum(x, b, dy, db)
    assert torch.equal(dx, ref_dx)
    assert ((db.double() - ref_db.double()).norm() / ref_db.double().norm()).item() < 1e-5
    # and against a torch fp32 reference of the op
    xf = (x.float() + b.float()).requires_grad_(True)
    torch.nn.functional.gelu(xf, approximate="tanh").backward(dy.float())
    assert rel(dx, xf.grad) < tol(dt)
    assert rel(db - 0.25, xf.grad.sum(0)) < tol(dt)


@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("dt", DT)
def test_embed_bwd_sorted(dt, gdt):
    """Deterministic sorted segment-sum embedding backward into a vocab shard's grad rows
    (bf16 or fp32), vs an fp64 index_add; repeated ids (runs) and ids of other shards."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(11)
    T, V, Hd, lo, Vl = 3000, 512, 4096 + 8 * 3, 128, 256
    ids = torch.randint(0, V, (T,), device="cuda")
    ids[:100] = 200  # a long run of one id
    dout = torch.randn(T, Hd, device="cuda").to(dt)
    base = torch.randn(Vl, Hd, device="cuda")
    grad = base.to(gdt).clone()
    K.embed_bwd_sorted(ids, dout, grad, vocab_lo=lo)
    ref = base.to(gdt).double().clone()
    mine = (ids >= lo) & (ids < lo + Vl)
    ref.index_add_(0, (ids[mine] - lo), dout[mine].double())
    assert rel(grad, ref) < (1e-6 if gdt == torch.float32 else 5e-3)
    untouched = torch.ones(Vl, dtype=torch.bool, device="cuda")
    untouched[(ids[mine] - lo).unique()] = False
    assert torch.equal(grad[untouched], base.to(gdt)[untouched])
    again = base.to(gdt).clone()
    K.embed_bwd_sorted(ids, dout, again, vocab_lo=lo)
    assert torch.equal(again, grad)  # deterministic


@pytest.mark.parametrize("V", [1001, 50304])
@pytest.mark.parametrize("dt", DT)
def test_xent_vocab_parallel_stages(dt, V):
    """Vocab-parallel cross-entropy as the tp>1 head runs it: stage 0 (row max per shard),
    max over shards, stage 1 (sum of exp + target logit per shard), sum over shards,
    stage 2 (loss + in-place gradient); vectorized (V/2 a multiple of 8) and scalar rows."""
    from paper_2504_21411_b200 import kernels as K
    torch.manual_seed(12)
    T = 257
    logits = (4 * torch.randn(T, V, device="cuda")).to(dt)
    labels = torch.randint(0, V, (T,), device="cuda")
    labels[3] = -100
    lr = logits.float().clone().requires_grad_(True)
    l_ref = torch.nn.functional.cross_entropy(lr, labels, reduction="none", ignore_index=-100)
    (l_ref.sum() / T).backward()
    loss = torch.empty(T, device="cuda")
    # fused single-launch path on the whole row (V = 1001: the scalar kernel)
    d = logits.clone()
    st = torch.empty(T, 3, device="cuda")
    K.xent(d, labels, st, 3, loss=loss, dlogits=d, grad_scale=1.0 / T)
    assert rel(loss, l_ref) < tol(dt)
    assert rel(d, lr.grad) < tol(dt) * 2
    if V % 2:
        return
    Vl = V // 2
    shards = [logits[:, :Vl].contiguous(), logits[:, Vl:].contiguous()]
    stats = [torch.empty(T, 3, device="cuda") for _ in shards]
    for sh, st, r in zip(shards, stats, range(2)):
        K.xent(sh, labels, st, 0, vocab_lo=r * Vl)
    mx = torch.maximum(stats[0][:, 0], stats[1][:, 0])
    for sh, st, r in zip(shards, stats, range(2)):
        st[:, 0] = mx
        K.xent(sh, labels, st, 1, vocab_lo=r * Vl)
    tot = stats[0][:, 1:3] + stats[1][:, 1:3]
    for sh, st, r in zip(shards, stats, range(2)):
        st[:, 1:3] = tot
        K.xent(sh, labels, st, 2, loss=loss, dlogits=sh, vocab_lo=r * Vl, grad_scale=1.0 / T)
    assert rel(loss, l_ref) < tol(dt)
    assert rel(torch.cat(shards, 1), lr.grad) < tol(dt) * 2
