"""Lowering of user equations to storage-indexed form.

Restates the parts of the reference's lowering the B200 backend depends on
(pkg/src/stencilc/lowering.py):

* ``affine_offset``: ``dim + k*unit`` -> integer k, opaque when the dim does
  not occur (lowering.py:199-233);
* ``indexify``: FD offsets divided out of every access (lowering.py:253-291);
* ``align_domain``: space indices shifted by halo+padding into storage
  coordinates (lowering.py:297-329);
* the data-space hull that caps the default ``*_M`` bounds so accesses stay
  in-allocation (lowering.py:486-514, operator.py:197-233).

Rebuilding through the canonical constructors re-sorts every sum and product
exactly as the reference does, which is why lowering is restated rather than
approximated: the lowered child order is the evaluation order.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from fractions import Fraction
from typing import Dict, List, Optional, Tuple

from ..symbolic.expr import (Access, Constant, Expr, Symbol, accesses_in, add,
                             call, children_of, evaluate, free_symbols, mul,
                             num, rebuild, substitute)
from ..symbolic.grid import Dimension, Equation, FunctionDecl


class LoweringError(ValueError):
    """Index expression the backend cannot lower."""


OPAQUE = object()


def affine_offset(index: Expr, dim_sym: Symbol, unit: Optional[Symbol]):
    """k such that index == dim + k*unit (or dim + k), OPAQUE if the dim
    symbol is absent."""
    if index == dim_sym:
        return 0
    if dim_sym.name not in free_symbols(index):
        return OPAQUE
    diff = add(index, mul(num(-1), dim_sym))
    rest = free_symbols(diff)
    allowed = {unit.name} if unit is not None else set()
    if not rest <= allowed:
        raise LoweringError("index %r is not affine in %s"
                            % (index, dim_sym.name))
    if not rest:
        if isinstance(diff, Constant) and \
                Fraction(diff.value).denominator == 1:
            return int(diff.value)
        raise LoweringError("non-integer index offset %r" % (diff,))
    v1 = evaluate(diff, {unit.name: 1.0})
    v2 = evaluate(diff, {unit.name: 2.0})
    v4 = evaluate(diff, {unit.name: 4.0})
    slope, icept = v2 - v1, 2 * v1 - v2
    if abs(icept + 4 * slope - v4) > 1e-9:
        raise LoweringError("index offset %r not linear in %s"
                            % (diff, unit.name))
    if abs(icept) > 1e-9 and abs(slope) > 1e-9:
        raise LoweringError("mixed index offset %r" % (diff,))
    k = slope if abs(slope) > 1e-9 else icept
    if abs(k - round(k)) > 1e-9:
        raise LoweringError("non-integer index offset %r" % (diff,))
    return int(round(k))


def _unit(decl: FunctionDecl, dim: Dimension) -> Optional[Symbol]:
    if dim.kind == "space":
        return None if decl.kind == "coordinates" else \
            decl.grid.spacing_of(dim)
    if dim.is_time:
        return decl.grid.step_symbol
    return None


def shift_of(decl: FunctionDecl, dim: Dimension) -> int:
    if dim.kind == "space" and decl.kind in ("function", "timefunction"):
        return decl.halo + decl.padding
    return 0


@dataclass
class LoweredEq:
    lhs: Access
    rhs: Expr
    is_increment: bool = False
    region: str = "domain"
    #: loop dims in order of appearance (time first when present)
    dims: Tuple[Dimension, ...] = ()
    #: per declaration: {storage-dim position: (lo, hi) hull incl. halo credit}
    dspace: Dict[int, Tuple[FunctionDecl, Dict[int, Tuple[int, int]]]] = \
        field(default_factory=dict)
    #: execution guards (root time dim name, factor): one per sub-sampled
    #: (conditional) dimension accessed, lhs first (reference
    #: lowering.py:246-291, Guard)
    guards: Tuple[Tuple[str, int], ...] = ()

    @property
    def is_dense(self) -> bool:
        return any(d.kind == "space" for d in self.dims)

    @property
    def has_time(self) -> bool:
        return any(d.is_time for d in self.dims)


def _indexify_access(acc: Access) -> Access:
    decl = acc.func
    if decl.kind == "temp":
        return acc
    if len(decl.dims) != len(acc.indices):
        raise LoweringError("arity mismatch accessing %s" % decl.name)
    out = []
    for dim, idx in zip(decl.dims, acc.indices):
        idx = _indexify(idx)
        if dim.kind == "conditional":
            if idx != dim.symbol:
                raise LoweringError("offsets on sub-sampled dimension %s "
                                    "unsupported" % dim.name)
            out.append(call("idiv", dim.parent.root.symbol, num(dim.factor)))
            continue
        k = affine_offset(idx, dim.symbol, _unit(decl, dim))
        out.append(idx if k is OPAQUE else add(dim.symbol, num(k)))
    return Access(decl, tuple(out))


def _indexify(e: Expr) -> Expr:
    if isinstance(e, Access):
        return _indexify_access(e)
    kids = children_of(e)
    return rebuild(e, [_indexify(c) for c in kids]) if kids else e


def _align_access(acc: Access) -> Access:
    decl = acc.func
    if decl.kind == "temp":
        return acc
    out = []
    for dim, idx in zip(decl.dims, acc.indices):
        idx = _align(idx)
        s = shift_of(decl, dim)
        out.append(add(idx, num(s)) if s else idx)
    return Access(decl, tuple(out))


def _align(e: Expr) -> Expr:
    if isinstance(e, Access):
        return _align_access(e)
    kids = children_of(e)
    return rebuild(e, [_align(c) for c in kids]) if kids else e


def _loop_dim(dim: Dimension) -> Dimension:
    return dim.root if dim.kind in ("stepping", "conditional") else dim


def access_offsets(acc: Access):
    """(storage pos, storage dim, loop dim, unaligned offset | OPAQUE)."""
    decl = acc.func
    out = []
    for pos, (dim, idx) in enumerate(zip(decl.dims, acc.indices)):
        if decl.kind == "temp":
            try:
                k = affine_offset(idx, dim.symbol, None)
            except LoweringError:
                k = OPAQUE
            out.append((pos, dim, dim, k))
            continue
        if dim.kind == "conditional":
            out.append((pos, dim, dim.parent.root, OPAQUE))
            continue
        loop = _loop_dim(dim)
        try:
            k = affine_offset(idx, Symbol(loop.name), None)
        except LoweringError:
            k = OPAQUE
        if k is not OPAQUE:
            k -= shift_of(decl, dim)
        out.append((pos, dim, loop, k))
    return out


def _all_accesses(lhs: Access, rhs: Expr) -> List[Access]:
    accs = [lhs] + _deep_accesses(rhs)
    for i in lhs.indices:
        accs += _deep_accesses(i)
    return accs


def _deep_accesses(e: Expr) -> List[Access]:
    out = []

    def walk(n):
        if isinstance(n, Access):
            out.append(n)
        for c in children_of(n):
            walk(c)
    walk(e)
    return out


def _analyze(low: LoweredEq) -> LoweredEq:
    order: List[Dimension] = []
    dspace: Dict[int, Tuple[FunctionDecl, Dict[int, Tuple[int, int]]]] = {}
    for acc in _all_accesses(low.lhs, low.rhs):
        decl = acc.func
        if decl.kind == "coordinates":
            continue
        for pos, dim, loop, k in access_offsets(acc):
            if k is not OPAQUE or dim.kind == "conditional":
                if loop not in order:
                    order.append(loop)
            else:
                for name in sorted(free_symbols(acc.indices[pos])):
                    if name.startswith("p_") and \
                            all(d.name != name for d in order):
                        order.append(Dimension(name, "sparse"))
            if decl.kind == "temp":
                continue
            slot = dspace.setdefault(id(decl), (decl, {}))[1]
            if k is OPAQUE:
                if dim.kind == "conditional":
                    lo, hi = 0, 0
                else:
                    continue
            elif dim.kind == "space":
                lo, hi = min(0, k + decl.halo), max(0, k - decl.halo)
            elif dim.kind == "stepping":
                lo, hi = 0, max(0, k)
            else:
                lo, hi = min(0, k), max(0, k)
            old = slot.get(pos)
            slot[pos] = (lo, hi) if old is None else \
                (min(old[0], lo), max(old[1], hi))
    # order of appearance, as the reference (lowering.py:410-435): an
    # equation writing a time-less function from time-indexed data
    # iterates time innermost
    return replace(low, dims=tuple(order), dspace=dspace)


def lower(eq: Equation, subs: Optional[dict] = None) -> LoweredEq:
    lhs = _indexify_access(eq.lhs)
    rhs = _indexify(eq.rhs)
    if subs:
        lhs = Access(lhs.func, tuple(substitute(i, subs) for i in lhs.indices))
        rhs = substitute(rhs, subs)
    low = LoweredEq(_align_access(lhs), _align(rhs), eq.is_increment,
                    eq.region)
    low = _analyze(low)
    guards = []
    for acc in [eq.lhs] + _deep_accesses(eq.rhs):
        if acc.func.kind == "temp":
            continue
        for dim in acc.func.dims:
            if dim.kind == "conditional":
                g = (dim.parent.root.name, dim.factor)
                if g not in guards:
                    guards.append(g)
    low.guards = tuple(guards)
    return low


def collect_functions(lowered: List[LoweredEq]) -> Dict[str, FunctionDecl]:
    """Every non-temp declaration touched (reference operator.py:91-102)."""
    out: Dict[str, FunctionDecl] = {}
    for eq in lowered:
        for acc in _all_accesses(eq.lhs, eq.rhs):
            if acc.func.kind != "temp":
                out.setdefault(acc.func.name, acc.func)
    return out
