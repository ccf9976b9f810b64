"""Block-shape autotuner: the reference's tuner
semantics (tests/test_iet.py:262-282 and test_acceptance.py:318-341 of the
reference) on the B200 backend, where a block shape sets the x planes per
CTA of the fused kernels and never changes results."""

import numpy as np
import pytest

import workloads
from paper_1807_03032_b200.backend import (BackendError, autotune,
                                           autotune_blocks,
                                           default_block_candidates)


def test_autotune_single_candidate():
    assert autotune_blocks(None, lambda c: 1.0, [{"x": 8}]) == {"x": 8}


def test_autotune_first_minimum_wins():
    times = {4: 2.0, 8: 1.0, 16: 1.0}
    got = autotune_blocks(None, lambda c: times[c["x"]],
                          [{"x": s} for s in (4, 8, 16)])
    assert got == {"x": 8}


def test_autotune_empty_candidates():
    with pytest.raises(BackendError):
        autotune_blocks(None, lambda c: 0.0, [])


def test_default_block_candidates_closed():
    cands = default_block_candidates(("x", "y", "z"))
    assert all(set(c) == {"x", "y", "z"} for c in cands)
    assert [c["x"] for c in cands] == [4, 8, 16, 32, 64]


@pytest.mark.gpu
@pytest.mark.parametrize("blk", [None, {"x": 4, "y": 64}, {"x": 16, "y": 16},
                                 {"x": 1, "y": 256}])
def test_yz_blocking_of_generated_kernels_vs_oracle(blk):
    """2D (generated NVRTC kernels): the block shape becomes the kernels'
    thread-block extents; every shape is bitwise the oracle."""
    import oracle
    import cases
    import paper_1807_03032_b200.symbolic as S
    from paper_1807_03032_b200.backend.operator import Operator
    case = cases.case_dict([c for c in cases.CASES
                            if c[0] == "ac2d_so4_f32_adv"][0])
    op = Operator(cases.build(S, case), mode=case["mode"], dtype=case["dtype"],
                  block=blk)
    bufs = op.allocate(case["nt"])
    cases.fill(bufs, case)
    ref = {k: type(v)(v.name, v.dtype, v.extents, data=v.data.copy())
           for k, v in bufs.items()}
    _, rep = op.apply(steps=case["nt"], buffers=bufs, dt=cases.dt_of(case))
    assert set([v for v in rep.values() if "dense_exec" in v][0]
               ["dense_exec"]) == {"generated"}
    out = oracle.apply(op, case["nt"], ref, dt=cases.dt_of(case))
    assert np.array_equal(bufs["u"].data, out["u"])
    assert np.array_equal(bufs["rec"].data, out["rec"])


@pytest.mark.gpu
def test_block_shape_never_changes_results():
    op0, bufs, dt, meta = workloads.config2(so=8, n=48, nbl=8, nt=8,
                                            nrec_side=8)
    rng = np.random.default_rng(5)
    inner = bufs["u"].data[0:2, 4:-4, 4:-4, 4:-4]
    inner[...] = rng.uniform(-1, 1, inner.shape).astype(np.float32)
    outs = []
    for blk in (None, {"x": 5}, {"x": 64}):
        op = type(op0)(op0.eqs, mode=op0.mode, dtype=op0.dtype, block=blk)
        b = {k: type(v)(v.name, v.dtype, v.extents, data=v.data.copy())
             for k, v in bufs.items()}
        op.apply(steps=meta["nt"], buffers=b, dt=dt)
        outs.append((b["u"].data, b["rec"].data))
    for u, r in outs[1:]:
        assert np.array_equal(u, outs[0][0]) and np.array_equal(r, outs[0][1])
    # and the shared result is the oracle's
    import oracle
    ref = oracle.apply(op0, meta["nt"], bufs, dt=dt)
    assert np.array_equal(outs[0][0], ref["u"])
    assert np.array_equal(outs[0][1], ref["rec"])


@pytest.mark.gpu
def test_autotune_self_consistent():
    """The returned shape attains the minimum the tuner itself measured
    (reference acceptance criterion 10)."""
    op, bufs, dt, meta = workloads.config2(so=8, n=96, nbl=8, nt=4,
                                           nrec_side=8)
    from paper_1807_03032_b200.backend.autotune import device_runner
    rec = {}
    base = device_runner(op.eqs, op.mode, op.dtype, 4, bufs, dt=dt)

    def runner(shape):
        rec[shape["x"]] = base(shape)
        return rec[shape["x"]]

    cands = [{"x": s} for s in (8, 16, 32, 64)]
    best = autotune_blocks(None, runner, cands)
    assert rec[best["x"]] <= min(rec.values())
    got = autotune(op.eqs, op.mode, op.dtype, steps=4, candidates=cands,
                   buffers=bufs, dt=dt)
    assert got in cands
