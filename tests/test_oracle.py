"""Pin the CPU model oracle (oracle/model_ref.py) against Hugging Face transformers
(golden file from tests/golden/make_model_golden.py, plus a live check when available)."""

import json
import math
from pathlib import Path

import pytest
import torch

from oracle import model_ref
from paper_2504_21411_b200.runtime.config import MODEL_PRESETS
from paper_2504_21411_b200.runtime.init import full_weights, param_shapes, synthetic_tokens

GOLD = json.loads((Path(__file__).parent / "golden" / "model_golden.json").read_text())

# oracle name -> HF name (grad norms are name-mapped; fused tensors compared by norm of parts)
def _hf_norms_to_oracle(cfg, hf):
    h, f = cfg.hidden, cfg.ffn
    out = {}
    if cfg.arch == "llama":
        out["embed.weight"] = hf["model.embed_tokens.weight"]
        out["final_norm.weight"] = hf["model.norm.weight"]
        out["lm_head.weight"] = hf["lm_head.weight"]
        for i in range(cfg.n_layers):
            p, q = f"layers.{i}.", f"model.layers.{i}."
            out[p + "qkv.weight"] = math.sqrt(sum(hf[q + f"self_attn.{n}_proj.weight"] ** 2
                                                  for n in "qkv"))
            out[p + "proj.weight"] = hf[q + "self_attn.o_proj.weight"]
            out[p + "gate_up.weight"] = math.hypot(hf[q + "mlp.gate_proj.weight"],
                                                   hf[q + "mlp.up_proj.weight"])
            out[p + "down.weight"] = hf[q + "mlp.down_proj.weight"]
            out[p + "attn_norm.weight"] = hf[q + "input_layernorm.weight"]
            out[p + "mlp_norm.weight"] = hf[q + "post_attention_layernorm.weight"]
    else:
        out["embed.weight"] = hf["transformer.wte.weight"]
        out["pos_embed.weight"] = hf["transformer.wpe.weight"]
        out["final_norm.weight"] = hf["transformer.ln_f.weight"]
        out["final_norm.bias"] = hf["transformer.ln_f.bias"]
        out["lm_head.weight"] = hf["lm_head.weight"]
        m = {"attn_norm": "ln_1", "mlp_norm": "ln_2", "qkv": "attn.c_attn",
             "proj": "attn.c_proj", "fc1": "mlp.c_fc", "fc2": "mlp.c_proj"}
        for i in range(cfg.n_layers):
            for a, b in m.items():
                for leaf in ("weight", "bias"):
                    out[f"layers.{i}.{a}.{leaf}"] = hf[f"transformer.h.{i}.{b}.{leaf}"]
    return out


@pytest.mark.parametrize("name", ["micro-llama", "micro-gpt"])
def test_oracle_matches_hf_golden(name):
    cfg = MODEL_PRESETS[name]
    w = full_weights(cfg, perturb=True)
    assert set(w) == set(model_ref.param_shapes(cfg)) == set(param_shapes(cfg))
    loss, grads = model_ref.loss_and_grads(cfg, w, synthetic_tokens(cfg, 2))
    gold = GOLD[name]
    assert abs(loss.item() - gold["loss"]) < 1e-10 * abs(gold["loss"])
    want = _hf_norms_to_oracle(cfg, gold["hf_grad_norms"])
    assert set(want) == set(grads)
    for n, g in grads.items():
        assert abs(g.norm().item() - want[n]) <= 1e-6 * max(want[n], 1e-12), n


def test_initial_loss_is_about_log_vocab():
    cfg = MODEL_PRESETS["micro-llama"]
    loss, _ = model_ref.loss_and_grads(cfg, full_weights(cfg), synthetic_tokens(cfg, 2))
    assert abs(loss.item() - math.log(cfg.vocab)) < 0.1


@pytest.mark.parametrize("name", ["micro-llama", "micro-gpt"])
def test_oracle_matches_live_hf(name):
    pytest.importorskip("transformers")
    import sys
    sys.path.insert(0, str(Path(__file__).parent / "golden"))
    from make_model_golden import hf_loss_and_grad_norms
    cfg = MODEL_PRESETS[name]
    w = full_weights(cfg, perturb=True, seed=99)
    tokens = synthetic_tokens(cfg, 2, seed=7)
    loss_hf, _ = hf_loss_and_grad_norms(cfg, w, tokens)
    loss, _ = model_ref.loss_and_grads(cfg, w, tokens)
    assert abs(loss.item() - loss_hf) < 1e-8 * abs(loss_hf)
