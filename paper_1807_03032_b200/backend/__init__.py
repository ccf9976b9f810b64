"""B200 backend: Operator (drop-in for reference backend/operator.py), buffers,
errors (reference backend/__init__.py:4-14)."""

from .buffers import BackendError, BoundsError, DataBuffer, allocate
from .operator import PASS_WORK, Operator, clear_cache
from .autotune import autotune, autotune_blocks, default_block_candidates

__all__ = ["BackendError", "BoundsError", "DataBuffer", "allocate",
           "Operator", "PASS_WORK", "clear_cache", "autotune",
           "autotune_blocks", "default_block_candidates"]
