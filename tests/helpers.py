"""Shared test helpers: golden fixtures and case runners."""

import hashlib
import json
import os

import numpy as np

import cases
import paper_1807_03032_b200.symbolic as S
from paper_1807_03032_b200.backend.operator import Operator

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden():
    with open(os.path.join(GOLDEN, "acoustic.json")) as f:
        return json.load(f)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make(case, mode=None, dtype=None):
    op = Operator(cases.build(S, case), mode=mode or case["mode"],
                  dtype=dtype or case["dtype"])
    bufs = op.allocate(case["nt"])
    cases.fill(bufs, case)
    return op, bufs


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb else 1.0)


CASE_IDS = [c[0] for c in cases.CASES]
CASES = {c[0]: cases.case_dict(c) for c in cases.CASES}
