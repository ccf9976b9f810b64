"""TTI: the operator authored with the reference API
(operators.tti_equations) is recognised for the fused kernel; the oracle
port reproduces the REAL reference bit for bit on it (goldens from
tests/golden/make_golden_tti.py); the GPU path agrees with the reference
within the north-star tolerance (rel-L2 <= 1e-5 wavefields, <= 1e-4 traces)."""

import hashlib
import json
import os

import numpy as np
import pytest

import tti_cases
import oracle
import paper_1807_03032_b200.symbolic as S
from paper_1807_03032_b200.backend.operator import Operator

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden():
    with open(os.path.join(GOLD, "tti.json")) as f:
        return json.load(f)


def _arrays(name):
    return np.load(os.path.join(GOLD, "arrays", name + ".npz"))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_tti_recognised_and_dse_bypassed():
    case = tti_cases.case_dict(tti_cases.CASES[0])
    op = Operator(tti_cases.build(S, case), dtype="f32")
    fused = [c for c in op.clusters if c.fused is not None]
    assert len(fused) == 1 and fused[0].fused[0] == "tti"
    roles = fused[0].fused[1]
    assert roles["theta"].name == "theta" and roles["m"].name == "m"


def test_tti_oracle_port_matches_reference_so4():
    case = tti_cases.case_dict(tti_cases.CASES[0])
    op = Operator(tti_cases.build(S, case), mode="advanced", dtype="f32",
                  fuse=False)
    trees = [repr((e.lhs, e.rhs)) for c in op.clusters for e in c.eqs]
    ref = _golden()["cases"][case["name"]]
    assert hashlib.sha256("\n".join(trees).encode()).hexdigest() == \
        ref["trees_sha"]
    bufs = op.allocate(case["nt"], pinned=False)
    tti_cases.fill(bufs, case)
    out = oracle.apply(op, case["nt"], bufs, dt=tti_cases.dt_of(case))
    for k in ("p", "r", "rec"):
        assert _sha(out[k]) == ref[k]["sha"], k


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.gpu
@pytest.mark.parametrize("row", tti_cases.CASES, ids=[c[0] for c in tti_cases.CASES])
def test_tti_gpu_vs_reference(row):
    case = tti_cases.case_dict(row)
    op = Operator(tti_cases.build(S, case), dtype="f32")
    bufs = op.allocate(case["nt"])
    tti_cases.fill(bufs, case)
    _, rep = op.apply(steps=case["nt"], buffers=bufs, dt=tti_cases.dt_of(case))
    assert [v for v in rep.values() if "fast_path" in v][0]["fast_path"]
    ref = _arrays(case["name"])
    for k in ("p", "r"):
        e32, e64 = _rel(bufs[k].data, ref[k]), _rel(bufs[k].data, ref[k + "64"])
        floor = _rel(ref[k], ref[k + "64"])
        assert e32 <= 1e-5 and e64 <= 1e-5, (k, e32, e64, floor)
    rec, r32 = bufs["rec"].data, ref["rec"]
    den = max(np.linalg.norm(r32), 1e-3 * np.abs(ref["rec64"]).max() *
              np.sqrt(r32.size))
    assert np.linalg.norm(rec - r32) / den <= 1e-4
