"""Golden loss/gradient vectors for the model oracle, computed by Hugging Face
``transformers`` (an independent implementation of GPT-2 / Llama) on the runtime's
deterministic logical weights.

    python tests/golden/make_model_golden.py      # writes tests/golden/model_golden.json

tests/test_oracle.py checks oracle/model_ref.py against this file (and, when
transformers is importable, against a live HF model).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2504_21411_b200.runtime.config import MODEL_PRESETS  # noqa: E402
from paper_2504_21411_b200.runtime.init import full_weights, synthetic_tokens  # noqa: E402


def hf_model(cfg, w):
    import transformers as tf
    h, f = cfg.hidden, cfg.ffn
    if cfg.arch == "llama":
        c = tf.LlamaConfig(vocab_size=cfg.vocab, hidden_size=h, intermediate_size=f,
                           num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.heads,
                           num_key_value_heads=cfg.heads, max_position_embeddings=cfg.seq_len,
                           rms_norm_eps=cfg.norm_eps, rope_theta=cfg.rope_theta,
                           tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
        m = tf.LlamaForCausalLM(c).double()
        sd = {"model.embed_tokens.weight": w["embed.weight"], "model.norm.weight":
              w["final_norm.weight"], "lm_head.weight": w["lm_head.weight"]}
        for i in range(cfg.n_layers):
            p, q = f"layers.{i}.", f"model.layers.{i}."
            qkv = w[p + "qkv.weight"]
            sd[q + "self_attn.q_proj.weight"] = qkv[:h]
            sd[q + "self_attn.k_proj.weight"] = qkv[h:2 * h]
            sd[q + "self_attn.v_proj.weight"] = qkv[2 * h:]
            sd[q + "self_attn.o_proj.weight"] = w[p + "proj.weight"]
            sd[q + "mlp.gate_proj.weight"] = w[p + "gate_up.weight"][:f]
            sd[q + "mlp.up_proj.weight"] = w[p + "gate_up.weight"][f:]
            sd[q + "mlp.down_proj.weight"] = w[p + "down.weight"]
            sd[q + "input_layernorm.weight"] = w[p + "attn_norm.weight"]
            sd[q + "post_attention_layernorm.weight"] = w[p + "mlp_norm.weight"]
    else:
        c = tf.GPT2Config(vocab_size=cfg.vocab, n_positions=cfg.seq_len, n_embd=h,
                          n_layer=cfg.n_layers, n_head=cfg.heads, n_inner=f,
                          activation_function="gelu_new", layer_norm_epsilon=cfg.norm_eps,
                          resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0,
                          tie_word_embeddings=False)
        m = tf.GPT2LMHeadModel(c).double()
        sd = {"transformer.wte.weight": w["embed.weight"], "transformer.wpe.weight":
              w["pos_embed.weight"], "transformer.ln_f.weight": w["final_norm.weight"],
              "transformer.ln_f.bias": w["final_norm.bias"], "lm_head.weight":
              w["lm_head.weight"]}
        for i in range(cfg.n_layers):
            p, q = f"layers.{i}.", f"transformer.h.{i}."
            sd[q + "ln_1.weight"] = w[p + "attn_norm.weight"]
            sd[q + "ln_1.bias"] = w[p + "attn_norm.bias"]
            sd[q + "attn.c_attn.weight"] = w[p + "qkv.weight"].t()
            sd[q + "attn.c_attn.bias"] = w[p + "qkv.bias"]
            sd[q + "attn.c_proj.weight"] = w[p + "proj.weight"].t()
            sd[q + "attn.c_proj.bias"] = w[p + "proj.bias"]
            sd[q + "ln_2.weight"] = w[p + "mlp_norm.weight"]
            sd[q + "ln_2.bias"] = w[p + "mlp_norm.bias"]
            sd[q + "mlp.c_fc.weight"] = w[p + "fc1.weight"].t()
            sd[q + "mlp.c_fc.bias"] = w[p + "fc1.bias"]
            sd[q + "mlp.c_proj.weight"] = w[p + "fc2.weight"].t()
            sd[q + "mlp.c_proj.bias"] = w[p + "fc2.bias"]
    missing, unexpected = m.load_state_dict({k: v.double().contiguous() for k, v in sd.items()},
                                            strict=False)
    missing = [k for k in missing if not k.endswith(("attn.bias", "masked_bias", "inv_freq"))]
    assert not missing and not unexpected, (missing, unexpected)
    m.eval()
    return m


def hf_loss_and_grad_norms(cfg, w, tokens):
    import torch.nn.functional as F
    m = hf_model(cfg, w)
    S = cfg.seq_len
    logits = m(input_ids=tokens[:, :S]).logits
    loss = F.cross_entropy(logits.reshape(-1, cfg.vocab), tokens[:, 1:S + 1].reshape(-1))
    loss.backward()
    norms = {n: p.grad.norm().item() for n, p in m.named_parameters() if p.grad is not None}
    return loss.item(), norms


def main():
    out = {}
    for name in ("micro-llama", "micro-gpt"):
        cfg = MODEL_PRESETS[name]
        w = full_weights(cfg, perturb=True)
        tokens = synthetic_tokens(cfg, 2)
        loss, norms = hf_loss_and_grad_norms(cfg, w, tokens)
        out[name] = {"loss": loss, "hf_grad_norms": norms}
    path = Path(__file__).with_name("model_golden.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote", path)


if __name__ == "__main__":
    main()
