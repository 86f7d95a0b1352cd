"""CPU restatement of GPT-2 / Llama-2 training numerics -- TEST INFRASTRUCTURE ONLY.

Parity status: UNPINNED against the reference (the reference repository has no model
code: SPEC.md:10).  The definitions are the standard ones and are cross-checked
against Hugging Face ``transformers`` on shared weights (tests/test_oracle.py):

GPT-2 block (pre-LN):  x += proj(attn(LN1(x))) ; x += fc2(gelu_tanh(fc1(LN2(x))))
  fused qkv with biases, learned absolute positions, final LN, untied LM head.
Llama-2 block:         x += proj(attn(rope(RMSNorm1(x)))) ; x += down(silu(gate)*up)
  RMSNorm eps 1e-5 (weight * x * rsqrt(mean(x^2)+eps)), rotate-half RoPE theta 1e4,
  no biases, final RMSNorm, untied LM head.
Causal softmax attention with scale 1/sqrt(head_dim); optional dropout of the attention
probabilities (cfg.attn_dropout) with the Philox4x32-10 mask of oracle/dropout_ref.py.  Loss = mean token
cross-entropy over all B*S positions of the global batch, labels = tokens shifted by
one (inputs tokens[:, :S], labels tokens[:, 1:S+1]).

``weights`` is a dict of full (unsharded) logical tensors named as in
``param_shapes`` below; the runtime slices the same logical tensors per rank.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def param_shapes(cfg) -> dict:
    """Logical parameter names -> shapes (documented contract shared with the runtime)."""
    h, f, V = cfg.hidden, cfg.ffn, cfg.vocab
    out = {"embed.weight": (V, h)}
    if cfg.arch == "gpt":
        out["pos_embed.weight"] = (cfg.seq_len, h)
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        if cfg.arch == "gpt":
            out.update({p + "attn_norm.weight": (h,), p + "attn_norm.bias": (h,),
                        p + "qkv.weight": (3 * h, h), p + "qkv.bias": (3 * h,),
                        p + "proj.weight": (h, h), p + "proj.bias": (h,),
                        p + "mlp_norm.weight": (h,), p + "mlp_norm.bias": (h,),
                        p + "fc1.weight": (f, h), p + "fc1.bias": (f,),
                        p + "fc2.weight": (h, f), p + "fc2.bias": (h,)})
        else:
            out.update({p + "attn_norm.weight": (h,), p + "qkv.weight": (3 * h, h),
                        p + "proj.weight": (h, h), p + "mlp_norm.weight": (h,),
                        p + "gate_up.weight": (2 * f, h), p + "down.weight": (h, f)})
    out["final_norm.weight"] = (h,)
    if cfg.arch == "gpt":
        out["final_norm.bias"] = (h,)
    out["lm_head.weight"] = (V, h)
    return out


def _rms(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _rope(x, theta):
    # x [B, S, H, D], rotate-half convention
    B, S, H, D = x.shape
    inv = 1.0 / theta ** (torch.arange(0, D, 2, dtype=torch.float32) / D)
    ang = torch.arange(S, dtype=torch.float32)[:, None] * inv[None, :]
    cos = ang.cos().to(x.dtype)[None, :, None, :]
    sin = ang.sin().to(x.dtype)[None, :, None, :]
    x1, x2 = x[..., : D // 2], x[..., D // 2:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def _attention(q, k, v, keep=None, p=0.0):
    # [B, S, H, D] -> [B, S, H, D], causal; keep: bool [B, H, S, S] dropout mask of the
    # attention probabilities (kept ones scaled by 1/(1-p)), oracle/dropout_ref.py
    B, S, H, D = q.shape
    qt, kt, vt = (t.transpose(1, 2) for t in (q, k, v))
    scores = qt @ kt.transpose(-1, -2) / math.sqrt(D)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool), diagonal=1)
    scores = scores.masked_fill(mask, float("-inf"))
    probs = torch.softmax(scores, dim=-1)
    if keep is not None:
        probs = probs * torch.as_tensor(keep).to(probs.dtype) / (1.0 - p)
    return (probs @ vt).transpose(1, 2)


def attention_keep_mask(cfg, B: int, layer: int, *, seed: int, step: int = 0):
    """The runtime's attention-dropout mask of decoder `layer` for a global batch of B
    sequences (Philox counter offset = (step << 16) | layer; sample / head indices global)."""
    from oracle.dropout_ref import keep_mask
    return keep_mask(B, cfg.seq_len, cfg.heads, cfg.attn_dropout, seed,
                     (step << 16) | layer)


def forward(cfg, w: dict, tokens: torch.Tensor, *, dropout_seed: int | None = None,
            dropout_step: int = 0):
    """Mean next-token loss of tokens [B, S+1] (int64) under weights ``w``; with
    cfg.attn_dropout > 0 and a dropout_seed, the attention probabilities are dropped with
    the runtime's Philox mask (attention_keep_mask)."""
    B = tokens.shape[0]
    S, h, H = cfg.seq_len, cfg.hidden, cfg.heads
    D = h // H
    ids, labels = tokens[:, :S], tokens[:, 1:S + 1]
    x = w["embed.weight"][ids]
    if cfg.arch == "gpt":
        x = x + w["pos_embed.weight"][:S][None]
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        if cfg.arch == "gpt":
            n = F.layer_norm(x, (h,), w[p + "attn_norm.weight"], w[p + "attn_norm.bias"],
                             cfg.norm_eps)
            qkv = n @ w[p + "qkv.weight"].t() + w[p + "qkv.bias"]
        else:
            n = _rms(x, w[p + "attn_norm.weight"], cfg.norm_eps)
            qkv = n @ w[p + "qkv.weight"].t()
        q, k, v = qkv.split(h, dim=-1)
        q, k, v = (t.reshape(B, S, H, D) for t in (q, k, v))
        if cfg.arch == "llama":
            q, k = _rope(q, cfg.rope_theta), _rope(k, cfg.rope_theta)
        p_drop = getattr(cfg, "attn_dropout", 0.0)
        keep = (attention_keep_mask(cfg, B, i, seed=dropout_seed, step=dropout_step)
                if p_drop > 0 and dropout_seed is not None else None)
        a = _attention(q, k, v, keep, p_drop).reshape(B, S, h)
        a = a @ w[p + "proj.weight"].t()
        if cfg.arch == "gpt":
            a = a + w[p + "proj.bias"]
        x = x + a
        if cfg.arch == "gpt":
            n = F.layer_norm(x, (h,), w[p + "mlp_norm.weight"], w[p + "mlp_norm.bias"],
                             cfg.norm_eps)
            m = F.gelu(n @ w[p + "fc1.weight"].t() + w[p + "fc1.bias"], approximate="tanh")
            m = m @ w[p + "fc2.weight"].t() + w[p + "fc2.bias"]
        else:
            n = _rms(x, w[p + "mlp_norm.weight"], cfg.norm_eps)
            g, u = (n @ w[p + "gate_up.weight"].t()).split(cfg.ffn, dim=-1)
            m = (F.silu(g) * u) @ w[p + "down.weight"].t()
        x = x + m
    if cfg.arch == "gpt":
        x = F.layer_norm(x, (h,), w["final_norm.weight"], w["final_norm.bias"], cfg.norm_eps)
    else:
        x = _rms(x, w["final_norm.weight"], cfg.norm_eps)
    logits = x @ w["lm_head.weight"].t()
    return F.cross_entropy(logits.reshape(-1, cfg.vocab), labels.reshape(-1))


def loss_and_grads(cfg, weights: dict, tokens: torch.Tensor, dtype=torch.float64, *,
                   dropout_seed: int | None = None, dropout_step: int = 0):
    """(loss, {name: grad}) for one fwd+bwd on CPU in ``dtype``."""
    w = {k: v.detach().to("cpu", dtype).clone().requires_grad_(True) for k, v in weights.items()}
    loss = forward(cfg, w, tokens.cpu(), dropout_seed=dropout_seed, dropout_step=dropout_step)
    loss.backward()
    return loss.detach(), {k: v.grad for k, v in w.items()}
