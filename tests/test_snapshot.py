"""Sub-sampled snapshots (reference lowering.py:
246-271 guards, iet.py:134-150 Conditional, test_backend.py:115-130):
``us[t/f] = u`` saved every f-th step inside the time loop, and an
imaging-condition accumulation ``img += us * u`` whose time loop the
reference schedules inside the space loops after the propagation. The
oracle port reproduces the real reference bit for bit (goldens from
tests/golden/make_golden_snapshot.py); the GPU reproduces the oracle bit
for bit."""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import snapshot_cases
import paper_1807_03032_b200.symbolic as S
from paper_1807_03032_b200.backend.operator import Operator

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
IDS = [c[0] for c in snapshot_cases.CASES]


def _golden():
    with open(os.path.join(GOLD, "snapshot.json")) as f:
        return json.load(f)["cases"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _op(case):
    return Operator(snapshot_cases.build(S, case), mode=case["mode"],
                    dtype=case["dtype"])


@pytest.mark.parametrize("row", snapshot_cases.CASES, ids=IDS)
def test_oracle_matches_reference(row):
    case = snapshot_cases.case_dict(row)
    ref = _golden()[case["name"]]
    op = _op(case)
    trees = [repr((e.lhs, e.rhs)) for c in op.clusters for e in c.eqs]
    assert hashlib.sha256("\n".join(trees).encode()).hexdigest() == \
        ref["trees_sha"]
    assert len(op.artifact.sections) == len(ref["points"])
    bufs = op.allocate(case["steps"], pinned=False)
    snapshot_cases.fill(bufs, case)
    out = oracle.apply(op, case["steps"], bufs, dt=snapshot_cases.DT)
    for k in ("u", "us", "img"):
        assert _sha(out[k]) == ref[k], k


def test_guards_and_time_inner_nest():
    case = snapshot_cases.case_dict(snapshot_cases.CASES[0])
    op = _op(case)
    snap = [c for c in op.clusters if c.eqs[-1].lhs.func.name == "us"][0]
    img = [c for c in op.clusters if c.eqs[-1].lhs.func.name == "img"][0]
    assert snap.guards == (("t", 3),) and snap.dims[0].is_time
    assert img.guards == (("t", 3),) and not img.dims[0].is_time


@pytest.mark.gpu
@pytest.mark.parametrize("row", snapshot_cases.CASES, ids=IDS)
def test_gpu_matches_reference(row):
    case = snapshot_cases.case_dict(row)
    ref = _golden()[case["name"]]
    op = _op(case)
    bufs = op.allocate(case["steps"])
    snapshot_cases.fill(bufs, case)
    _, rep = op.apply(steps=case["steps"], buffers=bufs, dt=snapshot_cases.DT)
    assert {k: v["points"] for k, v in rep.items()} == ref["points"]
    arrs = np.load(os.path.join(GOLD, "arrays", case["name"] + ".npz"))
    for k in ("u", "us", "img"):
        if _sha(bufs[k].data) != ref[k]:
            bad = np.argwhere(bufs[k].data != arrs[k])
            raise AssertionError("%s: %d points differ, first %s" %
                                 (k, len(bad), bad[:3]))
