"""Deterministic *global* parameter initialization and per-rank slicing.

Every logical (unsharded) tensor is drawn from its own generator seeded by
crc32(name) ^ seed, so every TP/DP/ZeRO/PP layout slices the same logical model
(SURVEY.md §8(d)): linear/embedding weights N(0, 0.02); norm weights 1 and biases 0
(``perturb=True`` draws norm weights 1+0.1N and biases 0.02N so parity tests see
non-trivial gradients through them).  ``param_shapes`` defines the names; the CPU
oracle consumes the same dict.
"""

from __future__ import annotations

import zlib

import torch

from .config import ModelConfig


def param_shapes(cfg: ModelConfig) -> dict:
    h, f, V = cfg.hidden, cfg.ffn, cfg.vocab
    out = {"embed.weight": (V, h)}
    if cfg.arch == "gpt":
        out["pos_embed.weight"] = (cfg.seq_len, h)
    for i in range(cfg.n_layers):
        out.update({f"layers.{i}.{k}": v for k, v in layer_param_shapes(cfg).items()})
    out["final_norm.weight"] = (h,)
    if cfg.arch == "gpt":
        out["final_norm.bias"] = (h,)
    out["lm_head.weight"] = (V, h)
    return out


def layer_param_shapes(cfg: ModelConfig) -> dict:
    h, f = cfg.hidden, cfg.ffn
    if cfg.arch == "gpt":
        return {"attn_norm.weight": (h,), "attn_norm.bias": (h,), "qkv.weight": (3 * h, h),
                "qkv.bias": (3 * h,), "proj.weight": (h, h), "proj.bias": (h,),
                "mlp_norm.weight": (h,), "mlp_norm.bias": (h,), "fc1.weight": (f, h),
                "fc1.bias": (f,), "fc2.weight": (h, f), "fc2.bias": (h,)}
    return {"attn_norm.weight": (h,), "qkv.weight": (3 * h, h), "proj.weight": (h, h),
            "mlp_norm.weight": (h,), "gate_up.weight": (2 * f, h), "down.weight": (h, f)}


def init_tensor(name: str, shape, *, seed: int = 1234, perturb: bool = False,
                device="cpu") -> torch.Tensor:
    gen = torch.Generator(device=device)
    gen.manual_seed((zlib.crc32(name.encode()) ^ seed) & 0x7FFFFFFF)
    leaf = name.rsplit(".", 2)
    is_norm = "norm" in name
    if name.endswith(".bias"):
        if perturb:
            return 0.02 * torch.randn(shape, generator=gen, device=device)
        return torch.zeros(shape, device=device)
    if is_norm:
        if perturb:
            return 1.0 + 0.1 * torch.randn(shape, generator=gen, device=device)
        return torch.ones(shape, device=device)
    del leaf
    return 0.02 * torch.randn(shape, generator=gen, device=device)


def full_weights(cfg: ModelConfig, *, seed: int = 1234, perturb: bool = False) -> dict:
    return {n: init_tensor(n, s, seed=seed, perturb=perturb) for n, s in param_shapes(cfg).items()}


def synthetic_tokens(cfg: ModelConfig, global_batch: int, *, seed: int = 1234,
                     device="cpu") -> torch.Tensor:
    """[global_batch, S+1] int64 tokens (SURVEY.md §8(d) synthetic inputs)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    return torch.randint(0, cfg.vocab, (global_batch, cfg.seq_len + 1), generator=gen,
                         device=device)
