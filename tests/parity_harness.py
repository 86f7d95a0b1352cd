"""Shared runtime-vs-oracle parity harness (single process or one rank of torchrun)."""

from __future__ import annotations

import torch

from oracle import model_ref
from paper_2504_21411_b200.planner.profiles import TrainingConfig
from paper_2504_21411_b200.runtime.config import MODEL_PRESETS, HybridConfig
from paper_2504_21411_b200.runtime.engine import construct_hybrid_parallel_model
from paper_2504_21411_b200.runtime.init import full_weights, synthetic_tokens


def rel(a, b) -> float:
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / (b.norm() + 1e-30)).item()


def oracle_after_steps(cfg, w, tokens, steps: int, optim):
    """CPU oracle: `steps` AdamW updates (torch.optim.AdamW, fp64), then loss + grads."""
    import torch
    params = {k: v.detach().to(torch.float64).clone().requires_grad_(True) for k, v in w.items()}
    opt = torch.optim.AdamW(params.values(), lr=optim.lr, betas=(optim.beta1, optim.beta2),
                            eps=optim.eps, weight_decay=optim.weight_decay)
    for _ in range(steps):
        opt.zero_grad()
        model_ref.forward(cfg, params, tokens.cpu()).backward()
        opt.step()
    return model_ref.loss_and_grads(cfg, {k: v.detach() for k, v in params.items()}, tokens,
                                    dtype=torch.float64)


def run_parity(name: str, hc: HybridConfig, dtype, *, grad_bytes: int = 4, seed: int = 1234,
               oracle_cache: dict | None = None, opt_steps: int = 0,
               oracle_dtype=torch.float64, attn_dropout: float = 0.0):
    """Returns (loss_err, {param: grad_err}) for this rank's stage params, after `opt_steps`
    optimizer steps (fused AdamW + ZeRO sharding) on the same batch.  attn_dropout > 0: the
    runtime and the oracle drop attention probabilities with the same Philox mask."""
    cfg = MODEL_PRESETS[name]
    if attn_dropout:
        if opt_steps:
            raise ValueError("dropout parity is checked on the first step")
        cfg = cfg.with_(attn_dropout=attn_dropout)
    w = full_weights(cfg, perturb=True, seed=seed)
    if dtype == torch.bfloat16:
        w = {k: v.bfloat16().float() for k, v in w.items()}
    tokens = synthetic_tokens(cfg, hc.global_batch, seed=seed)
    training = TrainingConfig(global_batch=hc.global_batch, bytes_per_grad=float(grad_bytes))
    from paper_2504_21411_b200.runtime.engine import OptimConfig
    optim = OptimConfig(lr=1e-3)
    model = construct_hybrid_parallel_model(cfg, hc, training=training, dtype=dtype, weights=w,
                                            optim=optim, seed=seed)
    for _ in range(opt_steps):
        model.train_step(tokens)
    loss = model.train_step(tokens, step_optimizer=False)
    grads = model.full_gradients()
    key = (name, hc.global_batch, seed, str(dtype), opt_steps, attn_dropout)
    if oracle_cache is not None and key in oracle_cache:
        ref_loss, ref_grads = oracle_cache[key]
    elif opt_steps:
        ref_loss, ref_grads = oracle_after_steps(cfg, w, tokens, opt_steps, optim)
    else:
        ref_loss, ref_grads = model_ref.loss_and_grads(
            cfg, w, tokens, dtype=oracle_dtype,
            dropout_seed=seed if cfg.attn_dropout > 0 else None)
        if oracle_cache is not None:
            oracle_cache[key] = (ref_loss, ref_grads)
    errs = {n: rel(g.float(), ref_grads[n]) for n, g in grads.items()}
    return abs(loss.item() - ref_loss.item()) / abs(ref_loss.item()), errs
