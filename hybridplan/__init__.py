"""Compatibility shim: ``import hybridplan`` resolves to the B200 build's planner.

Submodules (``hybridplan.search``, ``hybridplan.costmodel`` ...) alias the
modules of ``paper_2504_21411_b200.planner`` so code written against the
reference package runs unchanged.
"""

import sys as _sys

from paper_2504_21411_b200 import planner as _planner
from paper_2504_21411_b200.planner import *  # noqa: F401,F403
from paper_2504_21411_b200.planner import (cli, collectives, costmodel, errors, pipesim,
                                           profiles, search, serialize, strategy)

for _name in ("cli", "collectives", "costmodel", "errors", "pipesim", "profiles", "search",
              "serialize", "strategy"):
    _sys.modules[f"{__name__}.{_name}"] = getattr(_planner, _name)

__version__ = _planner.__version__
__all__ = list(_planner.__all__)
