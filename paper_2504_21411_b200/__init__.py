"""B200-native Galvatron runtime (arXiv 2504.21411 capabilities).

* ``planner``  -- drop-in ``hybridplan`` API: profiles, cost model, decision-tree +
  DP search, 1F1B simulator, CLI (bit-exact with the reference planner).
* ``runtime``  -- ``get_hybrid_parallel_configs`` / ``construct_hybrid_parallel_model``
  and the training engine: per-layer TP/SP/DP/ZeRO/recompute, reshard between
  layers, 1F1B pipeline, all on sm_100a kernels from ``csrc/`` via a C ABI.
* ``profiler`` -- measures this box (GEMM, NCCL bus bandwidth) into profile JSON.
"""

from . import planner  # noqa: F401

__version__ = "0.1.0"
