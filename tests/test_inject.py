"""Source injection (reference sparse.py:52-71 and the
point loop interpreter.py:173-186 / iet.py:234-245). Targets that collide
(sources sharing corners) are applied by a target-grouped kernel: one thread
per distinct target folds its increments in the reference's (point,
statement) order, so the result is bitwise the serial loop's while running
in parallel. Goldens: tests/golden/inject.json from the REAL reference
(tests/golden/make_golden_inject.py). SC_INJECT_ATOMIC=1 selects hardware
atomics (tolerance mode)."""

import hashlib
import json
import os

import numpy as np
import pytest

import inject_cases
import oracle
import paper_1807_03032_b200.symbolic as S
from paper_1807_03032_b200.backend.operator import Operator

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                    "inject.json")
NT = 8


def _gold():
    with open(GOLD) as f:
        return json.load(f)["cases"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _problem(nsrc, pinned=None):
    op = Operator(inject_cases.build(S, nsrc), dtype="f32")
    bufs = op.allocate(NT, pinned=pinned)
    inject_cases.fill(bufs)
    return op, bufs


def test_oracle_colliding_injection_matches_reference():
    """The oracle port applies colliding increments in the reference's
    point-outer order (pins the checker itself)."""
    op, bufs = _problem(1024, pinned=False)
    out = oracle.apply(op, NT, bufs, dt=inject_cases.DT)
    g = _gold()["collide_1024"]
    assert _sha(out["u"]) == g["u"] and _sha(out["rec"]) == g["rec"]


@pytest.mark.gpu
def test_colliding_injection_bitwise_and_fast():
    op, bufs = _problem(4096)
    _, rep = op.apply(NT, bufs, dt=inject_cases.DT)
    g = _gold()["collide_4096"]
    assert _sha(bufs["u"].data) == g["u"]
    assert _sha(bufs["rec"].data) == g["rec"]
    sec = [v for v in rep.values() if "stages" in v][0]
    inj = [v for k, v in sec["stages"].items() if k.startswith("sparse")][0]
    per_step_us = inj / NT * 1e6
    print("colliding injection, 4096 sources: %.1f us/step" % per_step_us)
    assert per_step_us < 50.0
    op.release()


@pytest.mark.gpu
def test_colliding_injection_atomic_tolerance(monkeypatch):
    monkeypatch.setenv("SC_INJECT_ATOMIC", "1")
    op, bufs = _problem(1024)
    ref = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
           for k, b in bufs.items()}
    op.apply(NT, bufs, dt=inject_cases.DT)
    out = oracle.apply(op, NT, ref, dt=inject_cases.DT)
    a = bufs["u"].data.astype(np.float64)
    b = out["u"].astype(np.float64)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5
    op.release()
