"""Host logic without a GPU: restated lowering/DSE reproduce the reference's
optimized trees (pinned by digests from the reference), plan construction,
fused-kernel selection, bounds and error conventions (dry plans)."""

import hashlib

import numpy as np
import pytest

import cases
from helpers import CASE_IDS, CASES, golden, make
from paper_1807_03032_b200.backend.buffers import BackendError, BoundsError


@pytest.mark.parametrize("name", CASE_IDS)
def test_optimized_trees_match_reference(name):
    op, _ = make(CASES[name])
    trees = [repr((e.lhs, e.rhs)) for c in op.clusters for e in c.eqs]
    digest = hashlib.sha256("\n".join(trees).encode()).hexdigest()
    assert digest == golden()["cases"][name]["trees_sha"]


@pytest.mark.parametrize("name", CASE_IDS)
def test_dry_plan(name):
    case = CASES[name]
    op, bufs = make(case)
    run = op.prepare(case["nt"], bufs, dry=True, dt=cases.dt_of(case))
    p = run.plan
    assert p.nstages == 3 and p.ndense == 1 and p.nsparse == 2
    fast = bool(run.fast_used)
    assert fast == (case["ndim"] == 3 and case["so"] > 2)
    assert p.sparse[0].kind == 0 and p.sparse[1].kind == 1
    assert bool(p.sparse[0].serial) == name.endswith("src4")


def test_bounds_and_unbound_symbols():
    case = CASES["ac3d_so4_f32_adv"]
    op, bufs = make(case)
    with pytest.raises(BoundsError):
        op.prepare(3, bufs, dry=True, dt=1.0, x_M=1000)
    with pytest.raises(BackendError):
        op.prepare(3, bufs, dry=True)          # dt unbound
    with pytest.raises(BoundsError):
        op.prepare(3, bufs, dry=True, dt=1.0, t_M=100)  # src/rec time axis


def test_default_params_caps():
    case = CASES["ac3d_so8_f32_adv"]
    op, _ = make(case)
    env = op.default_params(7)
    assert env["t_M"] == 6 and env["x_M"] == case["N"] - 1
    assert env["p_rec_M"] == case["nrec"] - 1


def test_fast_path_requires_canonical_names():
    """A field named below the oracle's temps reorders the Laplacian sums:
    the fused kernel must NOT be selected (the exact generic kernel runs)."""
    import workloads
    op = workloads.acoustic_operator((20, 20, 20), 10.0, 8, [(95., 95., 95.)],
                                     [(50., 50., 50.)], names=("a", "m", "damp"))
    bufs = op.allocate(4, pinned=False)
    run = op.prepare(4, bufs, dry=True, dt=1.0)
    assert not run.fast_used
    op2 = workloads.acoustic_operator((20, 20, 20), 10.0, 8, [(95., 95., 95.)],
                                      [(50., 50., 50.)])
    run2 = op2.prepare(4, op2.allocate(4, pinned=False), dry=True, dt=1.0)
    assert run2.fast_used


def test_cpu_has_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    case = CASES["ac1d_so4_f32_adv"]
    op, bufs = make(case)
    with pytest.raises(BackendError):
        op.apply(steps=2, buffers=bufs, dt=1.0)
