"""B200-native backend for the time-stepping loop behind the reference's
``Operator.apply`` (arXiv:1807.03032 / stencilc): isotropic acoustic and
TTI finite-difference operators, sparse source injection and receiver
interpolation, executed by hand-written sm_100a CUDA kernels through the C ABI
in include/stencil_b200.h.

The reference API is importable unchanged (``Grid``, ``FunctionDecl``,
``Eq``, ``solve_for``, ``inject``, ``interpolate``, ``Operator``); the
Devito-style names (``Function``, ``TimeFunction``, ``SparseTimeFunction``,
``solve``) live in ``facade``.
"""

from .symbolic import *  # noqa: F401,F403
from .symbolic import __all__ as _sym_all
from .backend import (BackendError, BoundsError, DataBuffer, Operator,
                      autotune, clear_cache)
from .facade import Function, SparseTimeFunction, TimeFunction, solve

__all__ = list(_sym_all) + ["BackendError", "BoundsError", "DataBuffer",
                            "Operator", "clear_cache", "autotune", "Function",
                            "TimeFunction", "SparseTimeFunction", "solve"]
