"""Operators built with the REFERENCE package run on the B200 backend
(backend/bridge.py). The reference is found at $REF, at
/root/reference (build container) or in baseline/_ref (the offline install
that travels to the GPU box: ``pip install --target baseline/_ref
/root/reference/pkg``)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_path():
    for p in (os.path.join(os.environ.get("REF", "/root/reference"), "pkg", "src"),
              os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "stencilc")):
            return p
    return None


REF = _ref_path()
needs_ref = pytest.mark.skipif(REF is None, reason="reference not present")


def _stencilc():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import stencilc.symbolic as RS
    from stencilc.backend.operator import Operator as RefOp
    return RS, RefOp


@needs_ref
def test_translated_operator_trees():
    import cases
    from paper_1807_03032_b200.backend.bridge import translate_operator
    RS, RefOp = _stencilc()
    case = cases.case_dict(cases.CASES[1])
    ref = RefOp(cases.build(RS, case), mode="advanced", dtype="f32")
    ours = translate_operator(ref)
    a = [repr((e.lhs, e.rhs)) for c in ref.artifact.clusters for e in c.eqs]
    b = [repr((e.lhs, e.rhs)) for c in ours.clusters for e in c.eqs]
    assert a == b


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("idx", [1, 8, 13], ids=["so8_f32", "so8_f64",
                                                  "src4_collide"])
def test_reference_operator_applied_on_gpu(idx):
    """A reference-built Operator applied through apply_reference_operator:
    the caller's reference DataBuffers hold, bit for bit, what the
    reference's own apply() produces (acoustic.json digests)."""
    import cases
    from helpers import golden, sha
    from paper_1807_03032_b200.backend.bridge import apply_reference_operator
    RS, RefOp = _stencilc()
    case = cases.case_dict(cases.CASES[idx])
    ref = RefOp(cases.build(RS, case), mode=case["mode"], dtype=case["dtype"])
    bufs = ref.allocate(case["nt"])
    cases.fill(bufs, case)
    out, report = apply_reference_operator(ref, case["nt"], bufs,
                                           dt=cases.dt_of(case))
    assert out is bufs
    gold = golden()["cases"][case["name"]]
    for k in ("u", "rec"):
        assert sha(bufs[k].data) == gold[k]["sha"], k
    assert any(v.get("fast_path") for v in report.values())


@needs_ref
@pytest.mark.gpu
def test_reference_tti_operator_applied_on_gpu():
    """The TTI system built with the reference's symbolic module (its so=4
    DSE compile takes ~10 s) runs through the bridge on the fused TTI
    kernels, within the north-star tolerance of the reference's arrays."""
    import tti_cases
    from paper_1807_03032_b200.backend.bridge import apply_reference_operator
    RS, RefOp = _stencilc()
    case = tti_cases.case_dict(tti_cases.CASES[0])
    ref = RefOp(tti_cases.build(RS, case), mode="advanced", dtype="f32")
    bufs = ref.allocate(case["nt"])
    tti_cases.fill(bufs, case)
    _, report = apply_reference_operator(ref, case["nt"], bufs,
                                         dt=tti_cases.dt_of(case))
    assert any(v.get("fast_path") for v in report.values())
    gold = np.load(os.path.join(ROOT, "tests", "golden", "arrays",
                                case["name"] + ".npz"))
    for k in ("p", "r"):
        a, b = bufs[k].data.astype(np.float64), gold[k].astype(np.float64)
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5, k
