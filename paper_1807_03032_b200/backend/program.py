"""Compile optimized trees into the exact operation sequences the kernels run.

The oracle evaluates a dense statement as whole-array numpy arithmetic
(reference interpreter.py:361-427) and every sparse statement point by point
through ``evaluate`` (expr.py:444-484, interpreter.py:224-240). In both
cases Python floats are *weak* scalars (NEP 50, numpy >= 2): they fold in
double precision among themselves and are rounded to the array dtype only
when they meet an array value. This module reproduces that typing to emit

* ``DenseProgram``: a straight-line register program (loads at fixed
  stencil offsets, ``a*k``/``a+k`` with pre-rounded constants, ``a*b``,
  ``a+b``, ``1/a``) -- the order of operations is exactly the oracle's;
* ``SparseProgram``: per corner, the ordered factor list of an injection or
  interpolation product and the corner summation order, plus the
  per-point index/weight tables evaluated with the oracle's float32
  semantics.

The kernels execute these sequences with round-to-nearest intrinsics and no
FMA contraction, so results are bitwise identical to the oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from ..symbolic.expr import (Access, Add, Call, Constant, Expr, Mul, Pow,
                             Symbol, children_of)
from .buffers import DTYPES, BackendError, BoundsError
from .lowering import OPAQUE, LoweredEq, access_offsets, affine_offset

# dense opcodes (mirrored in csrc/stencil_common.cuh)
OP_LOAD, OP_MULK, OP_ADDK, OP_MUL, OP_ADD, OP_RCP = range(6)


@dataclass
class Load:
    """Read of a dense function at a fixed offset from the update point."""

    func: str
    tshift: Optional[int]          # time offset (t + k), None for no time axis
    offs: Tuple[int, ...]          # storage offset minus loop index per dim
    tdiv: int = 1                  # >1: sub-sampled time index t // tdiv


@dataclass
class DenseProgram:
    ops: List[Tuple[int, int, int, int]] = field(default_factory=list)
    loads: List[Load] = field(default_factory=list)
    consts: List[float] = field(default_factory=list)
    out: Optional[int] = None
    target: Optional[Load] = None

    def signature(self):
        """Structure without constant values: two programs with equal
        signatures perform the same operations in the same order."""
        return (tuple(self.ops), tuple((l.func, l.tshift, l.offs, l.tdiv)
                                       for l in self.loads),
                len(self.consts), self.out,
                (self.target.func, self.target.tshift, self.target.offs,
                 self.target.tdiv))

    @property
    def nregs(self) -> int:
        return 1 + max([o[1] for o in self.ops] + [0])


class _DenseCompiler:
    def __init__(self, env: dict, dtype: str, stepping: Dict[str, object]):
        self.env = env
        self.np_t = DTYPES[dtype]
        self.prog = DenseProgram()
        self.vec: Dict[str, tuple] = {}
        self.nreg = 0
        self.load_ids: Dict[tuple, int] = {}
        self.const_ids: Dict[bytes, int] = {}

    def reg(self) -> int:
        self.nreg += 1
        return self.nreg - 1

    def const(self, v: float) -> int:
        r = self.np_t(v)               # weak scalar rounded at use
        key = r.tobytes()
        if key not in self.const_ids:
            self.const_ids[key] = len(self.prog.consts)
            self.prog.consts.append(float(r))
        return self.const_ids[key]

    def load(self, acc: Access) -> tuple:
        ld = point_load(acc)
        key = (ld.func, ld.tshift, ld.offs, ld.tdiv)
        if key not in self.load_ids:
            self.load_ids[key] = len(self.prog.loads)
            self.prog.loads.append(ld)
        r = self.reg()
        self.prog.ops.append((OP_LOAD, r, self.load_ids[key], 0))
        return ("a", r)

    def binop(self, op: str, a: tuple, b: tuple) -> tuple:
        if a[0] == "s" and b[0] == "s":
            return ("s", a[1] + b[1] if op == "+" else a[1] * b[1])
        if a[0] == "s":
            a, b = b, a                # + and * commute exactly in IEEE
        r = self.reg()
        if b[0] == "s":
            code = OP_ADDK if op == "+" else OP_MULK
            self.prog.ops.append((code, r, a[1], self.const(b[1])))
        else:
            code = OP_ADD if op == "+" else OP_MUL
            self.prog.ops.append((code, r, a[1], b[1]))
        return ("a", r)

    def ev(self, e: Expr) -> tuple:
        if isinstance(e, Constant):
            return ("s", float(e.value))
        if isinstance(e, Symbol):
            if e.name not in self.env:
                raise BackendError("unbound symbol %r" % e.name)
            return ("s", float(self.env[e.name]))
        if isinstance(e, Access):
            if e.func.kind == "temp" and not e.indices:
                if e.func.name not in self.vec:
                    raise BackendError("read of undefined scalar %s"
                                       % e.func.name)
                return self.vec[e.func.name]
            if e.func.kind not in ("function", "timefunction"):
                raise BackendError("unsupported access %r in a dense "
                                   "statement" % (e,))
            return self.load(e)
        if isinstance(e, (Add, Mul)):
            op = "+" if isinstance(e, Add) else "*"
            out = self.ev(e.children[0])
            for c in e.children[1:]:
                out = self.binop(op, out, self.ev(c))
            return out
        if isinstance(e, Pow):
            b = self.ev(e.base)
            if b[0] == "s":
                return ("s", b[1] ** e.exponent)
            if e.exponent == -1:
                r = self.reg()
                self.prog.ops.append((OP_RCP, r, b[1], 0))
                return ("a", r)
            if e.exponent == 2:        # numpy's fast path: square
                return self.binop("*", b, b)
            raise BackendError("array power %d has no exact kernel form"
                               % e.exponent)
        if isinstance(e, Call):
            args = [self.ev(a) for a in e.args]
            if all(a[0] == "s" for a in args) and e.name in ("min", "max"):
                return ("s", (min if e.name == "min" else max)(
                    a[1] for a in args))
            raise BackendError("call %s() has no exact kernel form" % e.name)
        raise BackendError("cannot compile %r" % (e,))


def point_load(acc: Access) -> Load:
    """Offsets of a dense access relative to the loop point, in storage
    units (reference interpreter.py:311-359 slice arithmetic)."""
    tshift, offs, tdiv = None, [], 1
    for pos, dim, loop, k in access_offsets(acc):
        if dim.kind == "conditional":   # us[t / f] (snapshots)
            tshift, tdiv = 0, dim.factor
            continue
        if k is OPAQUE:
            raise BackendError("non-affine access %r in dense statement"
                               % (acc,))
        if dim.kind in ("stepping", "time"):
            tshift = k
        elif dim.kind == "space":
            from .lowering import shift_of
            offs.append(k + shift_of(acc.func, dim))
        else:
            raise BackendError("unsupported dimension %s in %r"
                               % (dim.name, acc))
    return Load(acc.func.name, tshift, tuple(offs), tdiv)


def compile_dense(eqs: List[LoweredEq], env: dict, dtype: str
                  ) -> List[DenseProgram]:
    """One program per written dense function, scalar temps inlined."""
    comp = _DenseCompiler(env, dtype, {})
    progs = []
    for eq in eqs:
        f = eq.lhs.func
        if f.kind == "temp":
            if eq.lhs.indices:
                raise BackendError("array temporaries (%s) are not supported "
                                   "by the B200 backend" % f.name)
            comp.vec[f.name] = comp.ev(eq.rhs)
            continue
        if eq.is_increment:
            raise BackendError("dense increments are not supported")
        val = comp.ev(eq.rhs)
        if val[0] == "s":
            r = comp.reg()
            comp.prog.ops.append((OP_ADDK, r, -1, comp.const(val[1])))
            val = ("a", r)
        prog = comp.prog
        prog.out = val[1]
        prog.target = point_load(eq.lhs)
        progs.append(prog)
        comp.prog = DenseProgram()
        comp.nreg, comp.load_ids, comp.const_ids = 0, {}, {}
    for p in progs:
        p.ssa = list(p.ops)
        _allocate_registers(p)
    return progs


def program_trace(prog: DenseProgram) -> list:
    """Register-free form of a program: loads become their (function,
    time shift, offsets) key, constants their value, results the index of
    the producing operation. Equal traces = identical arithmetic."""
    out, ref = [], {}
    for i, (op, d, a, b) in enumerate(prog.ssa):
        if op == OP_LOAD:
            ld = prog.loads[a]
            ref[d] = ("ld", ld.func, ld.tshift, ld.offs) if ld.tdiv == 1 \
                else ("ld", ld.func, ld.tshift, ld.offs, ld.tdiv)
            continue
        if op in (OP_MULK, OP_ADDK):
            item = (op, ref[a] if a >= 0 else None, prog.consts[b])
        elif op in (OP_MUL, OP_ADD):
            item = (op, ref[a], ref[b])
        else:
            item = (op, ref[a], None)
        ref[d] = ("op", len(out))
        out.append(item)
    return out


def _allocate_registers(p: DenseProgram) -> None:
    """Linear-scan reuse: an SSA value's register frees after its last use."""
    last: Dict[int, int] = {}
    for i, (op, d, a, b) in enumerate(p.ops):
        if op in (OP_MULK, OP_ADDK, OP_RCP) and a >= 0:
            last[a] = i
        elif op in (OP_MUL, OP_ADD):
            last[a] = i
            last[b] = i
    last[p.out] = len(p.ops)
    free: List[int] = []
    phys: Dict[int, int] = {}
    nphys = 0
    new_ops = []
    for i, (op, d, a, b) in enumerate(p.ops):
        srcs = []
        if op in (OP_MULK, OP_ADDK, OP_RCP):
            if a >= 0:
                srcs = [a]
        elif op in (OP_MUL, OP_ADD):
            srcs = [a, b]
        pa = phys[a] if a >= 0 and op != OP_LOAD else a
        pb = phys[b] if op in (OP_MUL, OP_ADD) else b
        for s in set(srcs):
            if last.get(s) == i:
                free.append(phys[s])
        if free:
            pd = free.pop()
        else:
            pd = nphys
            nphys += 1
        phys[d] = pd
        new_ops.append((op, pd, pa, pb))
    p.ops = new_ops
    p.out = phys[p.out]


# -- sparse statements: per-point evaluate() with NEP 50 typing ---------------


class _Vec:
    """A per-point value: ``kind`` 'py' (Python float, double, uniform or
    per point as float64 array) or 'np' (numpy scalar of the operator
    dtype, per point as a dtype array)."""

    __slots__ = ("kind", "v")

    def __init__(self, kind, v):
        self.kind, self.v = kind, v


def _vop(op, a: _Vec, b: _Vec, np_t) -> _Vec:
    if a.kind == "py" and b.kind == "py":
        return _Vec("py", a.v + b.v if op == "+" else a.v * b.v)
    av = a.v if a.kind == "np" else np.asarray(a.v).astype(np_t)
    bv = b.v if b.kind == "np" else np.asarray(b.v).astype(np_t)
    return _Vec("np", (av + bv if op == "+" else av * bv).astype(np_t))


class SparseEvaluator:
    """Vectorised restatement of ``evaluate`` over all points of one sparse
    dimension (bit-identical to the per-point scalar loop: every numpy
    scalar op is an IEEE op in the dtype, every Python-float op is a double
    op)."""

    def __init__(self, env: dict, dtype: str, npoint: int,
                 buffers: Dict[str, np.ndarray], temps: Dict[str, _Vec],
                 pdim: str, pbase: int = 0, xoff: Dict[str, int] = None,
                 reads: Optional[list] = None):
        self.env = env
        # (function, index tuple, values) of every buffer gather, when the
        # caller wants to re-check later that the inputs are unchanged
        self.reads = reads
        self.np_t = DTYPES[dtype]
        self.n = npoint
        self.buffers = buffers
        self.temps = temps
        self.pdim = pdim
        self.pbase = pbase
        # dense arrays held as x windows: storage-x offset of plane 0
        self.xoff = xoff or {}
        # per-point values of subexpressions already evaluated (expressions
        # are immutable and compare structurally; the corner index and
        # weight expressions share their floor((c - o)/h) subtrees)
        self._memo: Dict[Expr, _Vec] = {}

    def index(self, e: Expr) -> np.ndarray:
        key = ("index", e)
        got = self._memo.get(key)
        if got is None:
            v = self.ev(e)
            x = np.broadcast_to(np.asarray(v.v, dtype=np.float64), (self.n,))
            got = self._memo[key] = np.rint(x).astype(np.int64)  # int(round(.))
        return got

    def ev(self, e: Expr) -> _Vec:
        if isinstance(e, (Constant, Symbol)):
            return self._ev(e)
        v = self._memo.get(e)
        if v is None:
            v = self._memo[e] = self._ev(e)
        return v

    def _ev(self, e: Expr) -> _Vec:
        np_t = self.np_t
        if isinstance(e, Constant):
            return _Vec("py", float(e.value))
        if isinstance(e, Symbol):
            if e.name == self.pdim:
                return _Vec("py", self.pbase + np.arange(self.n,
                                                         dtype=np.float64))
            if e.name not in self.env:
                raise BackendError("unbound symbol %r" % e.name)
            return _Vec("py", float(self.env[e.name]))
        if isinstance(e, Access):
            f = e.func
            if f.kind == "temp" and not e.indices:
                if f.name not in self.temps:
                    raise BackendError("read of undefined scalar %s" % f.name)
                return self.temps[f.name]
            if f.name not in self.buffers:
                raise BackendError("no buffer for %s" % f.name)
            buf = self.buffers[f.name]
            idx = []
            xpos = 1 if f.kind == "timefunction" else 0
            for pos, i in enumerate(e.indices):
                ii = self.index(i)
                if pos == 0 and getattr(f, "is_modulo_time", False):
                    ii = ii % f.time_dim.modulo
                if pos == xpos and f.name in self.xoff:
                    ii = ii - self.xoff[f.name]
                if ii.size and (ii.min() < 0 or ii.max() >= buf.shape[pos]):
                    bad = ii[(ii < 0) | (ii >= buf.shape[pos])][0]
                    raise BoundsError("%s index %d out of range [0, %d) along "
                                      "axis %d" % (f.name, bad, buf.shape[pos],
                                                   pos))
                idx.append(ii)
            vals = buf[tuple(idx)]
            if self.reads is not None:
                self.reads.append((f.name, tuple(idx), vals.copy()))
            return _Vec("np", vals.astype(np_t))
        if isinstance(e, Add):
            out = _Vec("py", 0.0)      # sum() starts from int 0
            for c in e.children:
                out = _vop("+", out, self.ev(c), np_t)
            return out
        if isinstance(e, Mul):
            out = _Vec("py", 1.0)
            for c in e.children:
                out = _vop("*", out, self.ev(c), np_t)
            return out
        if isinstance(e, Pow):
            b = self.ev(e.base)
            if b.kind == "py":
                if np.ndim(b.v):
                    return _Vec("py", np.array([x ** e.exponent for x in b.v]))
                return _Vec("py", b.v ** e.exponent)
            # numpy scalar power (libm pow/powf), evaluated per point
            out = np.array([x ** e.exponent for x in b.v], dtype=np_t)
            return _Vec("np", out)
        if isinstance(e, Call):
            args = [self.ev(a) for a in e.args]
            if e.name == "floor":
                a = args[0]
                return _Vec("py", np.floor(np.asarray(a.v, dtype=np.float64)))
            raise BackendError("call %s() in sparse statement unsupported"
                               % e.name)
        raise BackendError("cannot evaluate %r" % (e,))
