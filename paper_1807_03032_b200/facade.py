"""Devito-style names over the reference declaration model:
``Function``/``TimeFunction``/``SparseTimeFunction`` build ``FunctionDecl``
of kind function / timefunction / sparsetimefunction (reference
grid.py:122-185) and expose ``.dt``, ``.dt2``, ``.laplace``, ``.dx`` ...
(the suffixes the reference CLI parser maps, parser.py:221-248);
``solve(eq, target)`` is ``solve_for`` (fd.py:156-162) accepting either an
expression or an ``Eq``. ``Operator.apply(time_M=...)`` maps to ``t_M``.
"""

from __future__ import annotations

from .symbolic import fd as _fd
from .symbolic.expr import add, mul, num
from .symbolic.grid import Equation, FunctionDecl


class _Derivs:
    """Derivative properties shared by the Devito-style wrappers."""

    @property
    def dt(self):
        return _fd.dt(self)

    @property
    def dt2(self):
        return _fd.dt2(self)

    @property
    def laplace(self):
        return _fd.laplace(self)

    def _d(self, i, order):
        return _fd.derivative(self, self.grid.dimensions[i], self.space_order,
                              order)

    dx = property(lambda s: s._d(0, 1))
    dy = property(lambda s: s._d(1, 1))
    dz = property(lambda s: s._d(2, 1))
    dx2 = property(lambda s: s._d(0, 2))
    dy2 = property(lambda s: s._d(1, 2))
    dz2 = property(lambda s: s._d(2, 2))


class Function(FunctionDecl, _Derivs):
    def __init__(self, name, grid, space_order=2, padding=0):
        super().__init__(name, "function", grid, space_order=space_order,
                         padding=padding)


class TimeFunction(FunctionDecl, _Derivs):
    def __init__(self, name, grid, space_order=2, time_order=2, save=None,
                 time_dim=None, padding=0):
        super().__init__(name, "timefunction", grid, space_order=space_order,
                         time_order=time_order, save=save, time_dim=time_dim,
                         padding=padding)


class SparseTimeFunction(FunctionDecl):
    def __init__(self, name, grid, npoint, nt=None, coordinates=None):
        super().__init__(name, "sparsetimefunction", grid, npoint=npoint,
                         coordinates=coordinates)
        self.nt = nt

    def inject(self, field, expr):
        from .symbolic.sparse import inject
        return inject(self, field, expr)

    def interpolate(self, expr):
        from .symbolic.sparse import interpolate
        return interpolate(self, expr)


def solve(eq, target):
    """``solve(expr == 0 or Eq(lhs, rhs), target)`` -> expression."""
    if isinstance(eq, Equation):
        expr = add(eq.lhs, mul(num(-1), eq.rhs))
    else:
        expr = eq
    return _fd.solve_for(expr, target)
