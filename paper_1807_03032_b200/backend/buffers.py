"""Caller-owned host buffers and the backend's error types.

``DataBuffer`` keeps the reference's contract (interpreter.py:48-65): a
zero-initialised C-order numpy array per declared function, mutated in place
by ``Operator.apply``. Errors mirror interpreter.py:35-41.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

DTYPES = {"f32": np.float32, "f64": np.float64}


class BackendError(ValueError):
    """Malformed execution request (unbound symbol, bad dtype, unsupported
    equation, CUDA failure)."""


class BoundsError(IndexError):
    """An access would fall outside the allocated extents."""


@dataclass
class DataBuffer:
    name: str
    dtype: str
    extents: Tuple[int, ...]
    data: Optional[np.ndarray] = None

    def __post_init__(self):
        if self.dtype not in DTYPES:
            raise BackendError("bad dtype %r" % self.dtype)
        self.extents = tuple(int(e) for e in self.extents)
        if self.data is None:
            self.data = np.zeros(self.extents, DTYPES[self.dtype])
        elif tuple(self.data.shape) != self.extents:
            raise BackendError("data shape %r does not match extents %r"
                               % (self.data.shape, self.extents))


def allocate(decl, nt: Optional[int] = None, dtype: str = "f64") -> DataBuffer:
    return DataBuffer(decl.name, dtype, decl.storage_extents(nt))
