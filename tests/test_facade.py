"""Devito-style facade: ``SparseTimeFunction(nt=...)`` must
agree with the time axis the operator allocates (the reference sizes sparse
time axes by ``steps``, pkg/src/stencilc/backend/operator.py:185-190), and
``apply(time_M=...)`` without ``steps`` allocates ``time_M - time_m + 1``
steps. ``iet``/``source`` expose the compiled loop structure (reference
operator.py:160-166)."""

import pytest

from paper_1807_03032_b200 import (Eq, Function, Grid, Operator,
                                   SparseTimeFunction, Symbol, TimeFunction,
                                   solve)
from paper_1807_03032_b200.backend.buffers import BackendError


def _op(nt=None):
    g = Grid((20, 20, 20), extent=(190.,) * 3)
    u = TimeFunction("u", g, space_order=4)
    m = Function("m", g, space_order=4)
    src = SparseTimeFunction("src", g, npoint=1, nt=nt,
                             coordinates=[(95., 95., 95.)])
    rec = SparseTimeFunction("rec", g, npoint=1, nt=nt,
                             coordinates=[(50., 95., 30.)])
    d = Symbol("dt")
    return Operator([Eq(u.forward, solve(m.at * u.dt2 - u.laplace, u.forward))]
                    + src.inject(u.forward, src.at * d * d / m.at)
                    + rec.interpolate(u.at), dtype="f32")


def test_nt_must_match_allocated_steps():
    op = _op(nt=12)
    bufs = op.allocate(12, pinned=False)
    assert bufs["src"].data.shape == (12, 1)
    with pytest.raises(BackendError, match="nt=12"):
        op.allocate(10, pinned=False)


def test_steps_from_time_M_and_nt():
    op = _op(nt=12)
    assert op._steps(None, {"time_M": 9}) == 10
    assert op._steps(None, {"time_m": 2, "time_M": 9}) == 8
    assert op._steps(None, {}) == 12          # the declared nt
    assert op._steps(5, {"time_M": 9}) == 5   # explicit steps win
    assert _op()._steps(None, {}) == 1        # the reference's default


def test_iet_and_source():
    op = _op()
    iet = op.iet
    kinds = [n.kind for n in iet.walk()]
    assert kinds[0] == "Block" and "Section" in kinds and "Stage" in kinds
    stages = [n.name for n in iet.walk() if n.kind == "Stage"]
    assert stages == ["dense", "sparse-inject", "sparse-interpolate"]
    src = op.source
    assert "acoustic_kernel" in src and "sparse_interp_fast" in src
    assert "for t" in src
    assert op.dump_iet().startswith("Block kernel")
