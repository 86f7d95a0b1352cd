"""Single-GPU runtime parity vs the CPU oracle (loss and every parameter gradient).

Tolerances (north star): <= 1e-5 relative in fp32, <= 2e-2 relative in bf16
(relative L2 per tensor, ||x - ref|| / ||ref||).
"""

import pytest
import torch

from paper_2504_21411_b200.planner.strategy import ParallelStrategy
from paper_2504_21411_b200.runtime.config import MODEL_PRESETS, uniform_config

from parity_harness import run_parity

pytestmark = pytest.mark.gpu
S1 = ParallelStrategy(1, 1, 0, False, False)
S1R = ParallelStrategy(1, 1, 0, False, True)
CACHE: dict = {}


def test_tiny_gpt_fp32_config1():
    """BASELINE config 1: tiny GPT (4L, h512, 8 heads, s256, b8) fp32, 1 GPU."""
    hc = uniform_config(MODEL_PRESETS["tiny-gpt"], S1, microbatch=8, n_microbatches=1)
    lerr, errs = run_parity("tiny-gpt", hc, torch.float32, oracle_cache=CACHE)
    assert lerr <= 1e-5
    worst = max(errs.items(), key=lambda kv: kv[1])
    assert worst[1] <= 1e-5, worst


def test_tiny_gpt_fp32_microbatched_recompute():
    hc = uniform_config(MODEL_PRESETS["tiny-gpt"], S1R, microbatch=2, n_microbatches=4)
    lerr, errs = run_parity("tiny-gpt", hc, torch.float32, oracle_cache=CACHE)
    assert lerr <= 1e-5
    assert max(errs.values()) <= 1e-5, max(errs.items(), key=lambda kv: kv[1])


@pytest.mark.parametrize("name", ["micro-llama", "tiny-llama", "micro-gpt"])
def test_bf16_parity(name):
    cfg = MODEL_PRESETS[name]
    hc = uniform_config(cfg, S1, microbatch=2, n_microbatches=2)
    lerr, errs = run_parity(name, hc, torch.bfloat16, grad_bytes=4)
    assert lerr <= 2e-2
    worst = max(errs.items(), key=lambda kv: kv[1])
    assert worst[1] <= 2e-2, worst


@pytest.mark.parametrize("name", ["micro-llama", "micro-gpt"])
def test_bf16_parity_fused_activation_epilogues(name, monkeypatch):
    """Same bf16 parity with the SwiGLU / bias-GeLU GEMM-epilogue fusions forced on (the
    runtime enables them only for hidden >= 2048 / 4096, larger than these presets)."""
    from paper_2504_21411_b200.runtime import layers
    monkeypatch.setattr(layers, "FUSE_ACT_FWD_MIN_K", 0)
    monkeypatch.setattr(layers, "FUSE_ACT_BWD_MIN_K", 0)
    cfg = MODEL_PRESETS[name]
    hc = uniform_config(cfg, S1, microbatch=2, n_microbatches=2)
    lerr, errs = run_parity(name, hc, torch.bfloat16, grad_bytes=4)
    assert lerr <= 2e-2
    worst = max(errs.items(), key=lambda kv: kv[1])
    assert worst[1] <= 2e-2, worst


def test_llama_fp32_parity():
    cfg = MODEL_PRESETS["micro-llama"]
    hc = uniform_config(cfg, S1R, microbatch=1, n_microbatches=2)
    lerr, errs = run_parity("micro-llama", hc, torch.float32)
    assert lerr <= 1e-5
    assert max(errs.values()) <= 1e-5, max(errs.items(), key=lambda kv: kv[1])


def test_bf16_grad_buffers():
    """bytes_per_grad = 2 (the cost model default): bf16 gradient accumulation."""
    cfg = MODEL_PRESETS["micro-llama"]
    hc = uniform_config(cfg, S1, microbatch=1, n_microbatches=2)
    lerr, errs = run_parity("micro-llama", hc, torch.bfloat16, grad_bytes=2)
    assert lerr <= 2e-2 and max(errs.values()) <= 2e-2


@pytest.mark.parametrize("name,strategy", [("micro-llama", S1), ("micro-gpt", S1R)])
def test_fp32_parity_after_adamw_steps(name, strategy):
    """Two fused-AdamW steps (side-stream overlap) then loss/grads vs torch.optim.AdamW (fp64)."""
    cfg = MODEL_PRESETS[name]
    hc = uniform_config(cfg, strategy, microbatch=1, n_microbatches=2)
    lerr, errs = run_parity(name, hc, torch.float32, opt_steps=2)
    assert lerr <= 1e-4
    assert max(errs.values()) <= 1e-3, max(errs.items(), key=lambda kv: kv[1])
