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


def test_dropout_philox_known_answers():
    """oracle/dropout_ref.philox4x32_10 against the Random123 known-answer vectors for
    philox4x32-10 (the generator csrc/dropout.cuh implements)."""
    import numpy as np
    from oracle.dropout_ref import philox4x32_10
    kat = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
           ((0xffffffff,) * 4, (0xffffffff, 0xffffffff),
            (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
           ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
            (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]
    for ctr, key, want in kat:
        got = philox4x32_10(np.array(ctr, dtype=np.uint32), key)
        assert tuple(int(x) for x in got) == want


def test_dropout_mask_statistics_and_sharding_invariance():
    """Keep rate ~ 1-p; the mask of a (b0, h0)-offset block equals the matching slice of the
    global mask (why the runtime can shard attention over dp / tp / Ulysses)."""
    from oracle.dropout_ref import keep_mask
    full = keep_mask(4, 64, 6, 0.25, 99, 7)
    assert abs(full.mean() - 0.75) < 0.01
    part = keep_mask(2, 64, 3, 0.25, 99, 7, b0=1, h0=2, H_total=6)
    assert (part == full[1:3, 2:5]).all()
    assert not (keep_mask(4, 64, 6, 0.25, 99, 8) == full).all()
