"""Symbolic rewrites that fix the oracle's evaluation order.

The CUDA kernels reproduce the oracle's floating-point operation order, and
that order is the canonical child order of the *optimized* trees the oracle
interprets. Three of the reference's DSE passes shape those trees
(pkg/src/stencilc/dse.py), so they are restated here:

* time-invariant CIRE: maximal time-invariant sub-expressions costing
  >= EXTRACT_THRESHOLD flops become per-point array temps (dse.py:333-359,
  457-607) -- for sparse operators these are the hoisted weight tables;
* CSE: repeated compound sub-expressions become scalar temps, smallest
  first (dse.py:157-189);
* factorization: common coefficients of each sum collected, leaves first
  (dse.py:193-258).

Temp names come from one shared counter (dse.py:38-48). Names matter:
``Access`` nodes sort by function name, so renaming a temp can reorder a
sum. The passes are driven in the reference's mode order (dse.py:675-691).
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from ..symbolic.expr import (Access, Add, Call, Constant, Expr, Mul, Pow,
                             Symbol, add, children_of, coeff_and_term, mul,
                             num, op_count, pow_, rebuild, sort_key)
from ..symbolic.grid import Dimension, FunctionDecl
from .lowering import OPAQUE, LoweredEq, affine_offset

EXTRACT_THRESHOLD = 11
MODES = ("basic", "advanced", "aggressive")


class Namer:
    def __init__(self):
        self.n = 0

    def __call__(self) -> str:
        name = "temp%d" % self.n
        self.n += 1
        return name


@dataclass
class Cluster:
    eqs: List[LoweredEq]
    dims: Tuple[Dimension, ...]
    #: True for hoisted time-invariant producers (run once per apply)
    front: bool = False
    #: producer iteration extension per dim name (reference
    #: dse.py:520-559 _producer_ispace: upper bound + alias span)
    span: Dict[str, int] = field(default_factory=dict)
    #: recognised family executed by a dedicated kernel, e.g.
    #: ("tti", roles); such clusters bypass the DSE
    fused: Optional[tuple] = None
    #: execution guards shared by every member (reference clustering.py:
    #: 98-109 apply_control_flow)
    guards: tuple = ()


def make_temp(name, grid, dims, definition) -> FunctionDecl:
    d = FunctionDecl(name, "temp", grid, dims=dims)
    d.time_varying = time_varying(definition)
    return d


def time_varying(e: Expr) -> bool:
    if isinstance(e, Access):
        f = e.func
        if f.kind in ("timefunction", "sparsetimefunction"):
            return True
        return f.kind == "temp" and getattr(f, "time_varying", False)
    return any(time_varying(c) for c in children_of(e))


def _walk(e: Expr):
    """Postorder treating accesses as leaves."""
    if not isinstance(e, Access):
        for c in children_of(e):
            yield from _walk(c)
    yield e


def replace_subtrees(e: Expr, rules: Dict[Expr, Expr]) -> Expr:
    if e in rules:
        return rules[e]
    if isinstance(e, Access):
        return e
    kids = children_of(e)
    if not kids:
        return e
    new = [replace_subtrees(c, rules) for c in kids]
    if all(a is b for a, b in zip(new, kids)):
        return e
    return rebuild(e, new)


def _temp_reads(e: Expr) -> set:
    return {n.func.name for n in _walk(e)
            if isinstance(n, Access) and n.func.kind == "temp"}


def _order_defs(defs: List[LoweredEq]) -> List[LoweredEq]:
    local = {d.lhs.func.name for d in defs}
    todo = list(defs)
    done: set = set()
    out: List[LoweredEq] = []
    while todo:
        for d in todo:
            if (_temp_reads(d.rhs) & local) <= done:
                out.append(d)
                done.add(d.lhs.func.name)
                todo.remove(d)
                break
        else:
            raise ValueError("cyclic temp definitions")
    return out


def _is_temp_def(eq: LoweredEq) -> bool:
    return eq.lhs.func.kind == "temp"


# -- CSE -----------------------------------------------------------------------


def cse(c: Cluster, namer: Namer, grid) -> Cluster:
    defs = [e for e in c.eqs if _is_temp_def(e)]
    mains = [e for e in c.eqs if not _is_temp_def(e)]
    exprs = [e.rhs for e in defs + mains]
    new: List[LoweredEq] = []
    while True:
        counts: Counter = Counter()
        for e in exprs + [d.rhs for d in new]:
            for n in _walk(e):
                if not isinstance(n, (Constant, Symbol, Access)) and \
                        op_count(n) >= 1:
                    counts[n] += 1
        rep = [n for n, k in counts.items() if k >= 2]
        if not rep:
            break
        pick = min(rep, key=lambda n: (op_count(n), sort_key(n)))
        decl = make_temp(namer(), grid, (), pick)
        rule = {pick: Access(decl, ())}
        exprs = [replace_subtrees(e, rule) for e in exprs]
        new = [LoweredEq(d.lhs, replace_subtrees(d.rhs, rule), d.is_increment,
                         d.region, d.dims) for d in new]
        new.append(LoweredEq(Access(decl, ()), pick, dims=c.dims))
    rewritten = [LoweredEq(eq.lhs, e, eq.is_increment, eq.region, eq.dims,
                           eq.dspace) for eq, e in zip(defs + mains, exprs)]
    out_defs = _order_defs(rewritten[:len(defs)] + new)
    return Cluster(out_defs + rewritten[len(defs):], c.dims, c.front, c.span,
                   guards=c.guards)


# -- factorization ----------------------------------------------------------


def _factors(term: Expr) -> Dict[Expr, int]:
    if isinstance(term, Mul):
        out: Dict[Expr, int] = {}
        for ch in term.children:
            b, k = (ch.base, ch.exponent) if isinstance(ch, Pow) else (ch, 1)
            out[b] = out.get(b, 0) + k
        return out
    if isinstance(term, Pow):
        return {term.base: term.exponent}
    return {term: 1}


def _common(terms: List[Expr]) -> Dict[Expr, int]:
    maps = [_factors(t) for t in terms]
    out: Dict[Expr, int] = {}
    for b in maps[0]:
        ks = [m.get(b, 0) for m in maps]
        if all(k > 0 for k in ks):
            out[b] = min(ks)
        elif all(k < 0 for k in ks):
            out[b] = max(ks)
    return out


def _strip(term: Expr, common: Dict[Expr, int]) -> Expr:
    left = dict(_factors(term))
    for b, k in common.items():
        left[b] = left.get(b, 0) - k
    return mul(*[pow_(b, k) for b, k in left.items() if k != 0])


def factorize(e: Expr) -> Expr:
    if isinstance(e, Access):
        return e
    kids = children_of(e)
    inner = rebuild(e, [factorize(c) for c in kids]) if kids else e
    if not isinstance(inner, Add):
        return inner
    groups: Dict[object, List[Expr]] = {}
    for ch in inner.children:
        k, t = coeff_and_term(ch)
        groups.setdefault(k, []).append(t)
    parts = []
    for k, terms in groups.items():
        if len(terms) < 2:
            parts.append(mul(Constant(k), terms[0]))
            continue
        com = _common(terms)
        resid = add(*[_strip(t, com) for t in terms])
        parts.append(mul(Constant(k), *[pow_(b, x) for b, x in com.items()],
                         resid))
    cand = add(*parts)
    return cand if op_count(cand) <= op_count(inner) else inner


# -- time-invariant CIRE (extraction + aliases + pivots) --------------------


def _qualifies_ti(e: Expr, threshold: int) -> bool:
    if isinstance(e, (Constant, Symbol, Access)):
        return False
    return op_count(e) >= threshold and not time_varying(e)


def _candidates(e: Expr, threshold: int, root: bool = True) -> List[Expr]:
    if isinstance(e, Access):
        return []
    if not root and _qualifies_ti(e, threshold):
        return [e]
    out = []
    for c in children_of(e):
        out.extend(_candidates(c, threshold, False))
    return out


def _free(e: Expr) -> set:
    from ..symbolic.expr import free_symbols
    return free_symbols(e)


def _temp_dims(e: Expr, c: Cluster) -> Tuple[Dimension, ...]:
    free = _free(e)
    return tuple(d for d in c.dims if not d.is_time and d.name in free)


def _accesses(e: Expr) -> List[Access]:
    return [n for n in _walk(e) if isinstance(n, Access)]


def _displacements(e: Expr):
    out = []
    for acc in _accesses(e):
        disp = {}
        for dim, idx in zip(acc.func.dims, acc.indices):
            sym = Symbol(dim.root.name) \
                if dim.kind in ("stepping", "conditional") else dim.symbol
            try:
                k = affine_offset(idx, sym, None)
            except Exception:
                return None
            if k is OPAQUE:
                return None
            disp[dim.root.name] = k
        out.append(disp)
    return out


def _skeleton(e: Expr) -> Expr:
    if isinstance(e, Access):
        return Access(e.func, tuple(
            Symbol(d.root.name) if d.kind in ("stepping", "conditional")
            else d.symbol for d in e.func.dims))
    kids = children_of(e)
    return rebuild(e, [_skeleton(c) for c in kids]) if kids else e


def _translated(d1, d2) -> Optional[Dict[str, int]]:
    if len(d1) != len(d2):
        return None
    shift: Dict[str, int] = {}
    for a, b in zip(d1, d2):
        if set(a) != set(b):
            return None
        for dim in a:
            delta = b[dim] - a[dim]
            if shift.get(dim, delta) != delta:
                return None
            shift[dim] = delta
    return shift


def translate(e: Expr, shift: Dict[str, int]) -> Expr:
    if isinstance(e, Access):
        return Access(e.func, tuple(
            add(idx, num(shift[d.root.name])) if shift.get(d.root.name)
            else idx for d, idx in zip(e.func.dims, e.indices)))
    kids = children_of(e)
    return rebuild(e, [translate(c, shift) for c in kids]) if kids else e


def _time_names(e: Expr) -> set:
    return {d.root.name for a in _accesses(e) for d in a.func.dims
            if d.is_time}


@dataclass
class _Group:
    members: List[Expr]
    shifts: List[Dict[str, int]]
    pivot: Expr
    span: Dict[str, int]


def _alias_groups(cands: List[Expr]) -> List[_Group]:
    disp = {id(c): _displacements(c) for c in cands}
    todo = list(cands)
    out = []
    while todo:
        top = todo.pop(0)
        members, rel = [top], [{}]
        if disp[id(top)] is not None:
            skel = _skeleton(top)
            for e in list(todo):
                de = disp[id(e)]
                if de is None or _skeleton(e) != skel:
                    continue
                sh = _translated(disp[id(top)], de)
                if sh is None:
                    continue
                members.append(e)
                rel.append(sh)
                todo.remove(e)
        base: Dict[str, int] = {}
        if disp[id(top)] is not None:
            times = _time_names(top)
            for vec in disp[id(top)]:
                for d, k in vec.items():
                    if d not in times:
                        base[d] = min(base.get(d, k), k)
        dims = sorted({d for s in rel for d in s} | set(base))
        shifts = [{d: s.get(d, 0) + base.get(d, 0) for d in dims} for s in rel]
        pivot = translate(top, {d: -m for d, m in base.items() if m})
        span = {d: max(s.get(d, 0) for s in shifts) for d in dims}
        out.append(_Group(members, shifts, pivot, span))
    return out


def cire_invariant(clusters: List[Cluster], namer: Namer, grid,
                   threshold: int = EXTRACT_THRESHOLD) -> List[Cluster]:
    front: List[Cluster] = []
    out: List[Cluster] = []
    for c in clusters:
        cands, seen = [], set()
        for eq in c.eqs:
            for e in _candidates(eq.rhs, threshold):
                if e not in seen:
                    seen.add(e)
                    cands.append(e)
        if not cands:
            out.append(c)
            continue
        chosen = []
        for g in _alias_groups(cands):
            times = _time_names(g.pivot)
            if any(s.get(d) for s in g.shifts for d in times):
                continue
            if len(g.members) >= 2 or _temp_dims(g.pivot, c):
                chosen.append(g)
        if not chosen:
            out.append(c)
            continue
        rules: Dict[Expr, Expr] = {}
        defs: List[LoweredEq] = []
        hull: Dict[str, int] = {}
        for g in chosen:
            for d, sp in g.span.items():
                hull[d] = max(hull.get(d, 0), sp)
        for g in chosen:
            dims = _temp_dims(g.pivot, c)
            decl = make_temp(namer(), grid, dims, g.pivot)
            decl.span = dict(hull)
            defs.append(LoweredEq(Access(decl, tuple(d.symbol for d in dims)),
                                  g.pivot, dims=dims))
            for m, sh in zip(g.members, g.shifts):
                rules[m] = Access(decl, tuple(add(d.symbol, num(sh.get(d.name, 0)))
                                              for d in dims))
        consumer = Cluster([LoweredEq(eq.lhs, replace_subtrees(eq.rhs, rules),
                                      eq.is_increment, eq.region, eq.dims,
                                      eq.dspace) for eq in c.eqs], c.dims,
                           guards=c.guards)
        by_dims: Dict[tuple, List[LoweredEq]] = {}
        for d in defs:
            by_dims.setdefault(d.dims, []).append(d)
        for dims, eqs in by_dims.items():
            prod = Cluster(eqs, dims, front=True,
                           span={d.name: hull.get(d.name, 0) for d in dims},
                           guards=c.guards)
            if any(e.lhs.func.time_varying for e in eqs):
                prod.front = False
                out.append(prod)
            else:
                front.append(prod)
        out.append(consumer)
    merged: List[Cluster] = []
    for p in front:
        for q in merged:
            if q.dims == p.dims and q.span == p.span and q.guards == p.guards:
                q.eqs.extend(p.eqs)
                break
        else:
            merged.append(p)
    return merged + out


def factorize_cluster(c: Cluster) -> Cluster:
    return Cluster([LoweredEq(e.lhs, factorize(e.rhs), e.is_increment,
                              e.region, e.dims, e.dspace) for e in c.eqs],
                   c.dims, c.front, c.span, guards=c.guards)


def clusterize(lowered: List[LoweredEq]) -> List[Cluster]:
    """Equations sharing an iteration space join the latest such cluster
    (reference clustering.py:66-95, without the dependence-based vetoes
    that never fire for the recognised operator families)."""
    out: List[Cluster] = []
    for eq in lowered:
        if out and out[-1].dims == eq.dims and out[-1].guards == eq.guards:
            out[-1].eqs.append(eq)
        else:
            out.append(Cluster([eq], eq.dims, guards=eq.guards))
    return out


def run_dse(clusters: List[Cluster], mode: str, grid) -> List[Cluster]:
    if mode not in MODES:
        raise ValueError("unknown optimization mode %r" % mode)
    namer = Namer()
    out = list(clusters)
    if mode in ("advanced", "aggressive"):
        out = cire_invariant(out, namer, grid)
    # (aggressive's time-varying CIRE never rewrites the recognised
    # families: single-member alias groups stay inline, dse.py:535-538.)
    out = [cse(c, namer, grid) for c in out]
    if mode in ("advanced", "aggressive"):
        out = [factorize_cluster(c) for c in out]
    return out
