"""Selection of the fused acoustic kernel (csrc/acoustic.cu).

``acoustic_trace`` emits, operation by operation, what the CUDA kernel
computes for given role constants -- it is the kernel written out as a
program trace. An operator's compiled dense program is routed to the fused
kernel only when its trace (backend/program.py:program_trace) is *equal* to
this one, constants included; then the fused kernel is bitwise identical to
the exact generic program, and hence to the oracle. Anything else (other
equations, field names that reorder a sum, 1D/2D grids) runs the generic
program kernel, which is exact by construction.

Role constants are the scalar folds the oracle performs in double
(reference interpreter.py:383-388: symbols and constants are Python floats)
rounded once to the dtype when they meet an array.
"""

from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from ..symbolic.fd import centered_weights
from .buffers import DTYPES
from .program import OP_ADD, OP_ADDK, OP_MUL, OP_MULK, OP_RCP, DenseProgram

# role slots, mirrored in csrc/acoustic.cu
K_NEG1, K_HALF, K_T0, K_T1, K_MHALF, K_M2T1, K_DT2 = range(7)
K_C0, K_HSUM, K_H, K_CR, K_C0H, K_CRH, K_NUM = 7, 8, 9, 12, 21, 24, 48

FAST_FACT, FAST_BASIC = 1, 2


def group_radii(so: int) -> List[int]:
    """Coefficient-sorted group order of the Laplacian (matches
    ``group_radius`` in csrc/acoustic.cu)."""
    w = centered_weights(so, 2)
    return sorted(range(so // 2 + 1), key=lambda r: float(w[r]))


def role_constants(so: int, env: dict, damp: bool) -> List[float]:
    """Double-precision scalar folds, exactly as vec_eval forms them."""
    k = [0.0] * K_NUM
    dt = float(env["dt"])
    hs = [float(env["h_" + d]) ** -2 for d in "xyz"]
    t1 = dt ** -2
    k[K_NEG1] = -1.0
    k[K_HALF] = 0.5
    k[K_T0] = dt ** -1
    k[K_T1] = t1
    k[K_MHALF] = -0.5
    k[K_M2T1] = -2.0 * t1
    k[K_DT2] = dt ** 2
    w = centered_weights(so, 2)
    k[K_C0] = float(w[0])
    k[K_HSUM] = (hs[0] + hs[1]) + hs[2]
    for d in range(3):
        k[K_H + d] = hs[d]
        k[K_C0H + d] = float(w[0]) * hs[d]
    for r in range(1, so // 2 + 1):
        k[K_CR + r - 1] = float(w[r])
        for d in range(3):
            k[K_CRH + 3 * (r - 1) + d] = float(w[r]) * hs[d]
    return k


class _Trace:
    def __init__(self, np_t):
        self.items: list = []
        self.np_t = np_t

    def _push(self, item):
        self.items.append(item)
        return ("op", len(self.items) - 1)

    def mulk(self, a, v):
        return self._push((OP_MULK, a, float(self.np_t(v))))

    def mul(self, a, b):
        return self._push((OP_MUL, a, b))

    def add(self, a, b):
        return self._push((OP_ADD, a, b))

    def rcp(self, a):
        return self._push((OP_RCP, a, None))


def acoustic_trace(so: int, basic: bool, damp: bool, k: List[float],
                   names: Dict[str, str], dtype: str) -> list:
    """The fused kernel's operation sequence (acoustic.cu, acoustic_kernel)."""
    H = so // 2
    tr = _Trace(DTYPES[dtype])
    u, m, dmp = names["u"], names["m"], names.get("damp")

    def U(dx=0, dy=0, dz=0, ts=0):
        return ("ld", u, ts, (H + dx, H + dy, H + dz))
    c = (H, H, H)
    u0, um = U(), U(ts=-1)
    M = ("ld", m, None, c)
    D = ("ld", dmp, None, c) if damp else None

    # damped operators evaluate the 1/(...) factor before the Laplacian
    if damp:
        a = tr.add(tr.mulk(tr.mulk(D, k[K_HALF]), k[K_T0]),
                   tr.mulk(M, k[K_T1]))
        pn = tr.mulk(tr.rcp(a), k[K_NEG1])
    else:
        pn = tr.mulk(tr.mulk(tr.rcp(M), k[K_NEG1]), k[K_DT2])

    L = None
    for r in group_radii(so):
        if not basic:
            if r == 0:
                g = tr.mulk(tr.mulk(u0, k[K_C0]), k[K_HSUM])
            else:
                hx, hy, hz = (k[K_H + d] for d in range(3))
                s = tr.mulk(U(dx=-r), hx)
                s = tr.add(s, tr.mulk(U(dx=r), hx))
                s = tr.add(s, tr.mulk(U(dy=-r), hy))
                s = tr.add(s, tr.mulk(U(dy=r), hy))
                s = tr.add(s, tr.mulk(U(dz=-r), hz))
                s = tr.add(s, tr.mulk(U(dz=r), hz))
                g = tr.mulk(s, k[K_CR + r - 1])
            L = g if L is None else tr.add(L, g)
        else:
            if r == 0:
                L = tr.mulk(u0, k[K_C0H])
                L = tr.add(L, tr.mulk(u0, k[K_C0H + 1]))
                L = tr.add(L, tr.mulk(u0, k[K_C0H + 2]))
            else:
                kr = [k[K_CRH + 3 * (r - 1) + d] for d in range(3)]
                for (dx, dy, dz, kk) in ((-r, 0, 0, kr[0]), (r, 0, 0, kr[0]),
                                         (0, -r, 0, kr[1]), (0, r, 0, kr[1]),
                                         (0, 0, -r, kr[2]), (0, 0, r, kr[2])):
                    L = tr.add(L, tr.mulk(U(dx, dy, dz), kk))
    b1 = tr.mulk(L, k[K_NEG1])
    if damp:
        b2 = tr.mul(tr.mulk(tr.mulk(D, k[K_MHALF]), k[K_T0]), um)
        B = tr.add(b1, b2)
    else:
        B = b1
    inner = tr.add(tr.mulk(u0, k[K_M2T1]), tr.mulk(um, k[K_T1]))
    B = tr.add(B, tr.mul(M, inner))
    tr.mul(pn, B)
    return tr.items


def _normalise(trace: list) -> list:
    """Canonical op numbering: the kernel evaluates independent subtrees in
    a different order than the tree walk, which is harmless (each op's
    operands are fixed); compare the dataflow graph rooted at the result."""
    memo: Dict[int, tuple] = {}

    def node(ref):
        if ref is None or ref[0] == "ld":
            return ref
        i = ref[1]
        if i not in memo:
            op, a, b = trace[i]
            memo[i] = (op, node(a), node(b) if op in (OP_MUL, OP_ADD) else b)
        return memo[i]
    return node(("op", len(trace) - 1))


def match_acoustic(prog: DenseProgram, trace_user: list, so: int, env: dict,
                   names: Dict[str, str], dtype: str, has_damp: bool
                   ) -> Optional[tuple]:
    """(fast_kind, role constants) when the fused kernel computes exactly
    ``prog``; None otherwise."""
    try:
        k = role_constants(so, env, has_damp)
    except (KeyError, ZeroDivisionError, OverflowError):
        return None
    want = _normalise(trace_user)
    np_t = DTYPES[dtype]
    for basic, kind in ((False, FAST_FACT), (True, FAST_BASIC)):
        ref = acoustic_trace(so, basic, has_damp, k, names, dtype)
        if _normalise(ref) == want:
            return kind, [float(np_t(v)) for v in k]
    return None
