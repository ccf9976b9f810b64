"""A reference-built operator translates to identical optimized trees
(INTEGRATION.md §2); needs the reference tree (build container only)."""

import os
import sys

import pytest

REF = os.path.join(os.environ.get("REF", "/root/reference"), "pkg", "src")


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_translated_operator_trees():
    sys.path.insert(0, REF)
    import cases
    import stencilc.symbolic as RS
    from stencilc.backend.operator import Operator as RefOp
    from paper_1807_03032_b200.backend.bridge import translate_operator
    case = cases.case_dict(cases.CASES[1])
    ref = RefOp(cases.build(RS, case), mode="advanced", dtype="f32")
    ours = translate_operator(ref)
    a = [repr((e.lhs, e.rhs)) for c in ref.artifact.clusters for e in c.eqs]
    b = [repr((e.lhs, e.rhs)) for c in ours.clusters for e in c.eqs]
    assert a == b
