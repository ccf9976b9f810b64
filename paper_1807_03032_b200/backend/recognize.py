"""Recognition of operator families that have a fused sm_100a kernel whose
arithmetic is NOT the oracle's operation order (tolerance-level parity).

The acoustic family needs no recognizer: its fused kernel is selected by
program-trace equality (fastpath.py) and is bitwise exact. TTI is different:
its optimized tree (hundreds to thousands of operations per point after the
reference's DSE, which alone takes 10-941 s) is executed by
a hand-written kernel in its own FMA order. An equation pair is routed there
only if it is *structurally identical* to ``operators.tti_equations`` built
from the same declarations.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple

from ..symbolic.expr import Access, Call, Mul, Pow, Symbol, children_of
from ..symbolic.grid import Equation, FunctionDecl


def _funcs(e, kind: str, out: List[FunctionDecl]):
    if isinstance(e, Access):
        if e.func.kind == kind and all(e.func is not f for f in out):
            out.append(e.func)
    for c in children_of(e):
        _funcs(c, kind, out)


def _under_call(e, names, out: List[FunctionDecl], inside=False):
    if isinstance(e, Call) and e.name in names:
        inside = True
    if inside and isinstance(e, Access) and e.func.kind == "function":
        if all(e.func is not f for f in out):
            out.append(e.func)
    for c in children_of(e):
        _under_call(c, names, out, inside)


def _times_dt_power(e, power: int, out: List[FunctionDecl]):
    """Functions multiplied by dt**power somewhere in ``e``."""
    if isinstance(e, Mul):
        has = any(isinstance(c, Pow) and c.base == Symbol("dt") and
                  c.exponent == power for c in e.children)
        if has:
            for c in e.children:
                if isinstance(c, Access) and c.func.kind == "function" and \
                        all(c.func is not f for f in out):
                    out.append(c.func)
    for c in children_of(e):
        _times_dt_power(c, power, out)


def _is_forward(eq: Equation) -> bool:
    f = eq.lhs.func
    if f.kind != "timefunction" or eq.is_increment or not f.is_modulo_time:
        return False
    return eq.lhs == f.forward


def match_tti(eqs: List[Equation]) -> Optional[Tuple[int, int, Dict]]:
    """(index of the p equation, index of the r equation, role -> decl) when
    two of ``eqs`` are exactly ``tti_equations(p, r, m, damp, eps, delta,
    theta, phi)``."""
    from ..operators import tti_equations
    dense = [(i, e) for i, e in enumerate(eqs) if _is_forward(e)]
    if len(dense) != 2:
        return None
    (i, e1), (j, e2) = dense
    p, r = e1.lhs.func, e2.lhs.func
    so = p.space_order
    if so % 4 or r.space_order != so or p.grid.ndim != 3 or r.grid is not p.grid:
        return None
    fs: List[FunctionDecl] = []
    _funcs(e1.rhs, "function", fs)
    _funcs(e2.rhs, "function", fs)
    if len(fs) != 6:
        return None
    trig: List[FunctionDecl] = []
    _under_call(e1.rhs, ("sin", "cos"), trig)
    sq: List[FunctionDecl] = []
    _under_call(e1.rhs, ("sqrt",), sq)
    mdt: List[FunctionDecl] = []
    _times_dt_power(e1.rhs, -2, mdt)
    ddt: List[FunctionDecl] = []
    _times_dt_power(e1.rhs, -1, ddt)
    if len(trig) != 2 or len(sq) != 1 or len(mdt) != 1 or len(ddt) != 1:
        return None
    m, damp, delta = mdt[0], ddt[0], sq[0]
    rest = [f for f in fs if all(f is not g for g in trig + [m, damp, delta])]
    if len(rest) != 1:
        return None
    eps = rest[0]
    for th, ph in ((trig[0], trig[1]), (trig[1], trig[0])):
        want = tti_equations(p, r, m, damp, eps, delta, th, ph)
        if want[0] == e1 and want[1] == e2:
            return i, j, {"p": p, "r": r, "m": m, "damp": damp,
                          "epsilon": eps, "delta": delta, "theta": th,
                          "phi": ph}
    return None
