"""The library's multi-GPU data plane (include/stencil_b200.h sc_multi_*,
csrc/multi.cu): each rank's t loop -- boundary planes, NCCL ghost exchange on
a communication stream, interior planes -- captured as one CUDA graph
(sc_multi_run). One GPU is reachable here, so the GPU tests run a rank with
no neighbours through the native loop (the split schedule must be bitwise
the single-domain run) and the NCCL exchange against a one-rank
communicator whose 'neighbours' are the rank itself (checks the plane
offsets and the NCCL call path); the exchange between real neighbours is
covered by the host-side spec tests below and the gloo tests in
test_slab.py."""

import ctypes as C

import numpy as np
import pytest

import workloads
from paper_1807_03032_b200.backend import runtime as rt
from paper_1807_03032_b200.backend.slab import (SlabRank, attach_native,
                                                exchange_spec, step_loop)


def _problem(so=8, n=40, nbl=4, nt=8):
    op, bufs, dt, meta = workloads.config2(so=so, n=n, nbl=nbl, nt=nt,
                                           nrec_side=12)
    workloads.seed_interior(bufs, so, seed=7)
    return op, bufs, dt, meta


def test_exchange_struct_layout():
    assert C.sizeof(rt.ScExchange) == 76


@pytest.mark.parametrize("rank", [0, 1, 2])
def test_exchange_spec_of_a_middle_and_end_rank(rank):
    op, bufs, dt, meta = _problem()
    rk = SlabRank(op, bufs, rank, 3, meta["nt"], dry=True, overlap=True,
                  dt=dt)
    x = exchange_spec(rk)
    assert x.lo_peer == (rank - 1 if rank else -1)
    assert x.hi_peer == (rank + 1 if rank < 2 else -1)
    assert x.halo == 4 and x.slab == rk.b - rk.a
    assert x.nfields == 1 and x.field[0] == rk.run.field_ids["u"]
    # the split covers the slab once, in the run's local loop coordinates
    planes = []
    for k in range(x.nearly):
        planes += list(range(x.early[k][0], x.early[k][1] + 1))
    planes += list(range(x.interior[0], x.interior[1] + 1))
    sh = rk.run.xshift
    assert sorted(planes) == [p - sh for p in range(rk.a, rk.b)]
    assert x.n_early_points == rk.overlap["n_early"]


def _copy(bufs):
    return {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
            for k, b in bufs.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["acoustic", "tti"])
def test_native_slab_loop_bitwise(kind):
    """One rank, forced boundary/interior split, the whole loop in one
    graph through sc_multi_run: bitwise the single-domain apply."""
    if kind == "acoustic":
        op, bufs, dt, meta = _problem()
    else:
        op, bufs, dt, meta = workloads.config3(so=8, n=40, nbl=4, nt=6)
        workloads.seed_interior(bufs, 8, seed=11, fields=("p", "r"))
    single = _copy(bufs)
    op.apply(steps=meta["nt"], buffers=single, dt=dt)
    rk = SlabRank(op, bufs, 0, 1, meta["nt"], dt=dt, overlap="force")
    assert rk.overlap is not None
    attach_native(rk, None)
    step_loop(rk)
    out = _copy(bufs)
    rk.gather_into(out)
    for k in rk.written:
        assert np.array_equal(out[k].data, single[k].data), k
    rk.run.close()


@pytest.mark.gpu
def test_native_exchange_through_nccl_self_peers():
    """A one-rank NCCL communicator with both 'neighbours' set to the rank
    itself: NCCL pairs the sends and receives per peer in issue order, so
    the lower ghost planes receive the first H owned planes and the upper
    ghosts the last H -- exactly the offsets a real neighbour would fill."""
    import torch
    op, bufs, dt, meta = _problem()
    rk = SlabRank(op, bufs, 0, 1, meta["nt"], dt=dt)
    comm = rt.MultiComm(rt.multi_unique_id(), 0, 1)
    x = exchange_spec(rk, lo_peer=0, hi_peer=0)
    t = 2
    (_, v), = rk.slot_views(t)
    n, H = rk.b - rk.a, rk.H
    pattern = torch.arange(v.shape[0], device=v.device,
                           dtype=v.dtype).view(-1, 1, 1).expand_as(v)
    v.copy_(pattern + 0.5)
    prep = rk.run.prepared()
    prep.multi_exchange(comm, x, t, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = v[:, 0, 0].cpu().numpy()
    want = np.arange(v.shape[0]) + 0.5
    want[0:H] = np.arange(H, 2 * H) + 0.5          # lower ghosts <- first owned
    want[n + H:n + 2 * H] = np.arange(n, n + H) + 0.5   # upper <- last owned
    assert np.array_equal(got, want.astype(got.dtype))
    comm.close()
    rk.run.close()
