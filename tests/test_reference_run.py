"""``Operator.reference``: the reference's unoptimized per-equation executor
(pkg/src/stencilc/backend/operator.py:246-253 -> interpreter.py:493-549) --
no CSE, no factorization, no hoisting, no family kernels -- reproduced bit for
bit. Goldens: tests/golden/reference_run.json from the REAL reference
(tests/golden/make_golden_reference.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

import cases
import oracle
import snapshot_cases
import paper_1807_03032_b200.symbolic as S
from paper_1807_03032_b200.backend.operator import UNOPTIMIZED, Operator

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                    "reference_run.json")
with open(GOLD) as _f:
    REF = json.load(_f)["cases"]
ROWS = {r[0]: r for r in cases.CASES}
SROWS = {r[0]: r for r in snapshot_cases.CASES}


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _problem(name, pinned=None):
    if name in SROWS:
        case = snapshot_cases.case_dict(SROWS[name])
        op = Operator(snapshot_cases.build(S, case), mode=case["mode"],
                      dtype=case["dtype"])
        bufs = op.allocate(case["steps"], pinned=pinned)
        snapshot_cases.fill(bufs, case)
        return op, bufs, case["steps"], snapshot_cases.DT
    case = cases.case_dict(ROWS[name])
    op = Operator(cases.build(S, case), mode=case["mode"], dtype=case["dtype"])
    bufs = op.allocate(case["nt"], pinned=pinned)
    cases.fill(bufs, case)
    return op, bufs, case["nt"], cases.dt_of(case)


def test_unoptimized_schedule_is_one_nest_per_equation():
    op, _, _, _ = _problem("ac3d_so8_f32_adv", pinned=False)
    ref = Operator(op.eqs, mode=UNOPTIMIZED, dtype=op.dtype)
    assert len(ref.clusters) == len(op.eqs)
    assert [c.eqs[0].lhs for c in ref.clusters] == \
        [e.lhs for e in ref.artifact.lowered]
    # no temporaries anywhere: nothing was CSE'd or hoisted
    assert all(e.lhs.func.kind != "temp" for c in ref.clusters for e in c.eqs)


@pytest.mark.parametrize("name", ["ac3d_so4_f32_adv", "ac2d_so4_f32_adv",
                                  "ac3d_so8_f32_src4", "snap2d_so4_f3"])
def test_unoptimized_schedule_matches_reference_on_cpu(name):
    """The oracle port run over the unoptimized clusters reproduces the real
    reference's reference() (pins the schedule the GPU path executes)."""
    op, bufs, nt, dt = _problem(name, pinned=False)
    ref = Operator(op.eqs, mode=UNOPTIMIZED, dtype=op.dtype)
    out = oracle.apply(ref, nt, bufs, dt=dt)
    for k, h in REF[name].items():
        assert _sha(out[k]) == h, k


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(REF))
def test_gpu_reference_matches_reference(name):
    op, bufs, nt, dt = _problem(name)
    op.reference(steps=nt, buffers=bufs, dt=dt)
    for k, h in REF[name].items():
        assert _sha(bufs[k].data) == h, k
