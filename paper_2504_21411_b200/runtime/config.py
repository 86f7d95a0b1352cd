"""Model architecture configs and the per-layer hybrid-parallel configuration.

``get_hybrid_parallel_configs`` turns a planner ``Plan`` (reference
search.py:41-99 JSON) into the runtime's ``HybridConfig``: the per-layer
``ParallelStrategy`` list, pipeline degree, microbatch size and stage ranges.
``profile_for`` derives the planner's ``ModelProfile`` for an architecture so the
profiler -> search -> runtime flow uses one description of the model.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field, replace

from ..planner import profiles as _prof
from ..planner.errors import ValidationError
from ..planner.search import Plan
from ..planner.strategy import ParallelStrategy


@dataclass(frozen=True)
class ModelConfig:
    arch: str                # "gpt" (pre-LN, GeLU-tanh, biases, learned positions) | "llama"
    n_layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    seq_len: int
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0
    name: str = ""
    # dropout probability of the attention probabilities (softmax-dropout, north_star (1));
    # the BASELINE configs train with 0
    attn_dropout: float = 0.0

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def validate(self) -> None:
        if self.arch not in ("gpt", "llama"):
            raise ValidationError(f"unknown arch {self.arch!r}")
        if self.hidden % self.heads:
            raise ValidationError("hidden must be divisible by heads")
        if self.head_dim not in (64, 128):
            raise ValidationError("head_dim must be 64 or 128 (attention kernels)")
        if not 0.0 <= self.attn_dropout < 1.0:
            raise ValidationError("attn_dropout must be in [0, 1)")

    def layer_params(self) -> int:
        h, f = self.hidden, self.ffn
        if self.arch == "gpt":
            return 4 * h * h + 3 * h + h + 2 * h * f + f + h + 4 * h
        return 4 * h * h + 3 * h * f + 2 * h

    def total_params(self) -> int:
        emb = self.vocab * self.hidden + (self.seq_len * self.hidden if self.arch == "gpt" else 0)
        head = self.vocab * self.hidden + self.hidden * (2 if self.arch == "gpt" else 1)
        return self.n_layers * self.layer_params() + emb + head

    def train_flops_per_token(self) -> float:
        """6*L*P + 12*L*h*s + 6*h*V (non-causal count; matches the cost model's
        flops_per_token = 2P, flops_per_token_sq = 4h, bwd = 2x fwd)."""
        L, h, s, V = self.n_layers, self.hidden, self.seq_len, self.vocab
        return 6.0 * L * self.layer_params() + 12.0 * L * h * s + 6.0 * h * V

    def train_flops_per_token_causal(self) -> float:
        """Same with the causal half of the attention score/PV FLOPs only (the work the
        causal attention kernels actually do): 6*L*P + 6*L*h*s + 6*h*V."""
        L, h, s, V = self.n_layers, self.hidden, self.seq_len, self.vocab
        return 6.0 * L * self.layer_params() + 6.0 * L * h * s + 6.0 * h * V

    def with_(self, **kw) -> "ModelConfig":
        return replace(self, **kw)


MODEL_PRESETS = {
    # BASELINE.json configs (SURVEY.md §8 notation C1..C5)
    "tiny-gpt": ModelConfig("gpt", 4, 512, 8, 2048, 8192, 256, name="tiny-gpt"),
    "gpt2-medium": ModelConfig("gpt", 24, 1024, 16, 4096, 50304, 1024, name="gpt2-medium"),
    "gpt-1.3b": ModelConfig("gpt", 24, 2048, 16, 8192, 50304, 2048, name="gpt-1.3b"),
    "llama2-7b": ModelConfig("llama", 32, 4096, 32, 11008, 32000, 4096, name="llama2-7b"),
    "llama2-13b": ModelConfig("llama", 40, 5120, 40, 13824, 32000, 32768, name="llama2-13b"),
    # small configs used by the parity tests
    "tiny-llama": ModelConfig("llama", 4, 512, 8, 1408, 8192, 256, name="tiny-llama"),
    "micro-llama": ModelConfig("llama", 2, 256, 4, 704, 1024, 128, name="micro-llama"),
    "micro-gpt": ModelConfig("gpt", 2, 256, 4, 1024, 1024, 128, name="micro-gpt"),
    # head_dim 128 (the Llama-2-7B/13B head): exercises the RoPE-fused QKV GEMM epilogue
    # and galv_attn_bwd_rope exactly as the headline runs them
    "micro-llama128": ModelConfig("llama", 2, 256, 2, 704, 1024, 256, name="micro-llama128"),
    "mini-llama128": ModelConfig("llama", 2, 512, 4, 1408, 1024, 256, name="mini-llama128"),
    # one decoder layer at Llama-2-7B width and sequence length (h4096, 32x128, ffn 11008,
    # s4096, V 32000): the production shapes of every kernel of the headline step
    "llama2-7b-1l": ModelConfig("llama", 1, 4096, 32, 11008, 32000, 4096, name="llama2-7b-1l"),
}


def profile_for(cfg: ModelConfig, *, bytes_per_act: float = 2.0) -> _prof.ModelProfile:
    """Planner ModelProfile of the decoder layers (embedding/head are not planned layers,
    as in the reference: SPEC.md:98)."""
    if cfg.arch == "gpt" and cfg.ffn == 4 * cfg.hidden:
        return _prof.synth_transformer_profile(cfg.n_layers, cfg.hidden, cfg.seq_len)
    if cfg.arch == "gpt":
        raise ValidationError("gpt profiles assume ffn = 4*hidden")
    return _prof.synth_llama_profile(cfg.n_layers, cfg.hidden, cfg.seq_len, cfg.ffn,
                                     bytes_per_act=bytes_per_act)


@dataclass(frozen=True)
class HybridConfig:
    """What the runtime needs from a Plan: per-layer strategies and the pipeline layout."""

    pp: int
    microbatch: int
    n_microbatches: int
    stage_ranges: tuple
    layer_strategies: tuple
    predicted_iteration_time: float = float("nan")
    # "megatron": sp=True layers run Megatron-SP (weights tp-sharded, AG/RS around GEMMs).
    # "ulysses": sp=True layers run DeepSpeed-Ulysses over the same rank group: weights
    #   replicated in the group (grads all-reduced over it), tokens sequence-sharded, two
    #   all-to-alls (sequence <-> heads) around attention.  Runtime extension outside the
    #   reference strategy space: the cost model's param/tp memory term
    #   does not describe it.
    sp_mode: str = "megatron"

    @property
    def global_batch(self) -> int:
        return self.microbatch * self.n_microbatches

    @property
    def devices_per_stage(self) -> int:
        s = self.layer_strategies[0]
        return s.tp * s.dp

    @property
    def world_size(self) -> int:
        return self.pp * self.devices_per_stage

    def stage_of_layer(self, li: int) -> int:
        for i, (a, b) in enumerate(self.stage_ranges):
            if a <= li < b:
                return i
        raise ValidationError(f"layer {li} not in any stage")

    def validate(self, cfg: ModelConfig) -> None:
        if len(self.layer_strategies) != cfg.n_layers:
            raise ValidationError("one strategy per decoder layer required")
        width = self.devices_per_stage
        if self.sp_mode not in ("megatron", "ulysses"):
            raise ValidationError(f"unknown sp_mode {self.sp_mode!r}")
        for i, s in enumerate(self.layer_strategies):
            s.validate(width)
            if self.microbatch % s.dp:
                raise ValidationError(f"layer {i}: microbatch not divisible by dp")
            if cfg.heads % s.tp or cfg.ffn % s.tp:
                raise ValidationError(f"layer {i}: tp={s.tp} does not divide heads/ffn")
            tokens = self.microbatch * cfg.seq_len // s.dp
            if s.sp and tokens % s.tp:
                raise ValidationError(f"layer {i}: sp needs tokens divisible by tp")


def get_hybrid_parallel_configs(plan, model_cfg: ModelConfig | None = None, *,
                                sp_mode: str = "megatron", model_profile=None, cluster=None,
                                training=None, transitions: bool = True) -> HybridConfig:
    """Plan object, Plan dict, or path to a Plan JSON -> HybridConfig (validated).

    With the profiles the plan was searched under (``model_profile`` / ``cluster`` /
    ``training``), the plan is first re-checked by ``validate_plan`` (reference
    search.py:823-913: partition, degrees, divisibility, re-costed time within 1e-9
    relative, stage peaks within the memory budget) and refused with ``InvalidPlan``
    on any violation -- a plan produced under another profile, or one that no longer
    fits, does not run silently."""
    from ..planner.errors import InvalidPlan
    if isinstance(plan, (str, bytes)) or hasattr(plan, "__fspath__"):
        with open(plan, "r", encoding="utf-8") as fh:
            plan = json.load(fh)
    if isinstance(plan, dict):
        plan = Plan.from_dict(plan)
    if not isinstance(plan, Plan):
        raise ValidationError("expected a Plan, plan dict, or plan path")
    given = [x is not None for x in (model_profile, cluster, training)]
    if any(given) and not all(given):
        raise ValidationError("plan validation needs model_profile, cluster and training")
    if all(given):
        from ..planner.search import validate_plan
        problems = validate_plan(plan, model_profile, cluster, training,
                                 transitions=transitions)
        if problems:
            raise InvalidPlan(problems)
    hc = HybridConfig(pp=plan.pp, microbatch=plan.microbatch,
                      n_microbatches=plan.n_microbatches,
                      stage_ranges=tuple(tuple(r) for r in plan.stage_ranges),
                      layer_strategies=tuple(plan.layer_strategies),
                      predicted_iteration_time=plan.predicted_iteration_time, sp_mode=sp_mode)
    if model_cfg is not None:
        hc.validate(model_cfg)
    return hc


def uniform_config(cfg: ModelConfig, strategy: ParallelStrategy, *, pp: int = 1,
                   microbatch: int, n_microbatches: int) -> HybridConfig:
    """Hand-built config: the same strategy on every layer, near-equal stage split."""
    from ..planner.search import near_equal_split
    return HybridConfig(pp=pp, microbatch=microbatch, n_microbatches=n_microbatches,
                        stage_ranges=near_equal_split(cfg.n_layers, pp),
                        layer_strategies=(strategy,) * cfg.n_layers)
