"""B200 hybrid-parallel training runtime (the paper's "Runtime", absent from the reference).

Entry points named after the paper:
  get_hybrid_parallel_configs(plan, model_cfg)  -> HybridConfig
  construct_hybrid_parallel_model(model_cfg, hybrid_config, ...) -> HybridParallelModel
"""

from .config import MODEL_PRESETS, HybridConfig, ModelConfig, get_hybrid_parallel_configs  # noqa
from .engine import HybridParallelModel, OptimConfig, construct_hybrid_parallel_model  # noqa
