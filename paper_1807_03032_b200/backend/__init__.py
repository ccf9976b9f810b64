"""B200 backend: Operator (drop-in for reference backend/operator.py), buffers,
errors (reference backend/__init__.py:4-14)."""

from .buffers import BackendError, BoundsError, DataBuffer, allocate
from .operator import PASS_WORK, Operator, clear_cache

__all__ = ["BackendError", "BoundsError", "DataBuffer", "allocate",
           "Operator", "PASS_WORK", "clear_cache"]
