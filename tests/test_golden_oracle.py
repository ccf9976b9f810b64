"""The CPU oracle (oracle/) reproduces the REAL reference bit for bit on
every golden case (fixtures from tests/golden/make_golden.py): final
wavefield, receiver traces and the hoisted sparse index/weight tables."""

import pytest

import oracle
from helpers import CASE_IDS, CASES, golden, make, sha
import cases


@pytest.mark.parametrize("name", CASE_IDS)
def test_oracle_matches_reference(name):
    case = CASES[name]
    ref = golden()["cases"][name]
    op, bufs = make(case)
    out = oracle.apply(op, case["nt"], bufs, dt=cases.dt_of(case))
    checked = 0
    for k, v in ref.items():
        if k in ("u", "rec") or k.startswith("temp"):
            assert sha(out[k]) == v["sha"], k
            checked += 1
    assert checked >= 2
