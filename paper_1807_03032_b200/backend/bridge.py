"""Run an operator built with the REFERENCE package on the B200 backend.

``apply_reference_operator(ref_op, steps, buffers, **params)`` is the
maintainer-side shim of INTEGRATION.md §2: it re-declares the reference
operator's functions with this package's declarations (same names, kinds,
orders, coordinates), rebuilds its equations node by node through the
canonical constructors (which reproduce the reference's trees), and applies
the result to the caller's ``DataBuffer.data`` arrays in place.

Only duck typing is used (class names and attributes of the reference's
``symbolic.expr`` / ``symbolic.grid``), so the reference is not imported.
"""

from __future__ import annotations

from typing import Dict

from ..symbolic import expr as E
from ..symbolic.grid import Dimension, Equation, FunctionDecl, Grid
from .buffers import BackendError, DataBuffer
from .operator import Operator


class _Translator:
    def __init__(self):
        self.grids: Dict[int, Grid] = {}
        self.funcs: Dict[int, FunctionDecl] = {}

    def grid(self, g) -> Grid:
        key = id(g)
        if key not in self.grids:
            self.grids[key] = Grid(g.shape, g.extent, g.origin)
        return self.grids[key]

    def dim(self, d) -> Dimension:
        parent = self.dim(d.parent) if d.parent is not None else None
        return Dimension(d.name, d.kind, parent, d.factor, d.modulo)

    def func(self, f) -> FunctionDecl:
        key = id(f)
        if key in self.funcs:
            return self.funcs[key]
        if f.kind in ("coordinates", "temp"):
            raise BackendError("cannot translate %s declaration %s"
                               % (f.kind, f.name))
        g = self.grid(f.grid)
        td = None
        if f.kind == "timefunction" and f.time_dim is not None and \
                f.time_dim.kind == "conditional":
            td = self.dim(f.time_dim)
        new = FunctionDecl(f.name, f.kind, g, space_order=f.space_order,
                           time_order=f.time_order, save=f.save,
                           npoint=f.npoint,
                           coordinates=getattr(f, "coordinate_values", None),
                           time_dim=td,
                           padding=f.padding)
        self.funcs[key] = new
        if f.kind == "sparsetimefunction":
            self.funcs[id(f.coordinates)] = new.coordinates
        return new

    def expr(self, e):
        kind = type(e).__name__
        if kind == "Constant":
            return E.Constant(e.value)
        if kind == "Symbol":
            return E.Symbol(e.name)
        if kind == "Access":
            f = e.func
            decl = self.funcs.get(id(f))
            if decl is None:
                decl = self.func(f)
            return E.Access(decl, tuple(self.expr(i) for i in e.indices))
        if kind == "Add":
            return E.add(*[self.expr(c) for c in e.children])
        if kind == "Mul":
            return E.mul(*[self.expr(c) for c in e.children])
        if kind == "Pow":
            return E.pow_(self.expr(e.base), e.exponent)
        if kind == "Call":
            return E.call(e.name, *[self.expr(a) for a in e.args])
        raise BackendError("cannot translate expression node %r" % (e,))

    def equation(self, eq) -> Equation:
        return Equation(self.expr(eq.lhs), self.expr(eq.rhs), eq.region,
                        eq.is_increment)


def _deep_funcs(e, out):
    if type(e).__name__ == "Access":
        out.append(e.func)
    for attr in ("children", "args", "indices"):
        for c in getattr(e, attr, ()) or ():
            _deep_funcs(c, out)
    if type(e).__name__ == "Pow":
        _deep_funcs(e.base, out)


def translate_operator(ref_op) -> Operator:
    tr = _Translator()
    funcs: list = []
    for eq in ref_op.eqs:
        _deep_funcs(eq.lhs, funcs)
        _deep_funcs(eq.rhs, funcs)
    for f in funcs:                 # sparse functions register coordinates
        if f.kind not in ("coordinates", "temp"):
            tr.func(f)
    eqs = [tr.equation(eq) for eq in ref_op.eqs]
    return Operator(eqs, mode=ref_op.mode, dtype=ref_op.dtype,
                    subs=None, name=ref_op.name)


def apply_reference_operator(ref_op, steps: int = 1, buffers=None, **params):
    """Reference ``Operator.apply`` semantics on the GPU: ``buffers`` (the
    reference's DataBuffer dict) is updated in place."""
    op = translate_operator(ref_op)
    if buffers is None:
        buffers = ref_op.allocate(steps)
    ours = {k: DataBuffer(k, b.dtype, b.extents, data=b.data)
            for k, b in buffers.items()}
    _, report = op.apply(steps, ours, **params)
    for k, b in ours.items():
        if k not in buffers:         # hoisted tables, like the reference
            buffers[k] = b
    return buffers, report
