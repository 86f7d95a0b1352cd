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


def run_parity(name: str, hc: HybridConfig, dtype, *, grad_bytes: int = 4, seed: int = 1234,
               oracle_cache: dict | None = None):
    """Returns (loss_err, {param: grad_err}) for this rank's stage params."""
    cfg = MODEL_PRESETS[name]
    w = full_weights(cfg, perturb=True, seed=seed)
    if dtype == torch.bfloat16:
        w = {k: v.bfloat16().float() for k, v in w.items()}
    tokens = synthetic_tokens(cfg, hc.global_batch, seed=seed)
    training = TrainingConfig(global_batch=hc.global_batch, bytes_per_grad=float(grad_bytes))
    model = construct_hybrid_parallel_model(cfg, hc, training=training, dtype=dtype, weights=w)
    loss = model.train_step(tokens, step_optimizer=False)
    grads = model.full_gradients()
    key = (name, hc.global_batch, seed, str(dtype))
    if oracle_cache is not None and key in oracle_cache:
        ref_loss, ref_grads = oracle_cache[key]
    else:
        ref_loss, ref_grads = model_ref.loss_and_grads(cfg, w, tokens, dtype=torch.float64)
        if oracle_cache is not None:
            oracle_cache[key] = (ref_loss, ref_grads)
    errs = {n: rel(g.float(), ref_grads[n]) for n, g in grads.items()}
    return abs(loss.item() - ref_loss.item()) / abs(ref_loss.item()), errs
