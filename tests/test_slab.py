"""x-slab decomposition: decomposed runs are bitwise equal
to the single-domain run.

* CPU, world_size 2 over gloo (torch.distributed): each rank computes its
  slab with the oracle port (test infrastructure stands in for the kernels)
  and exchanges ghost planes with gloo point-to-point -- this exercises the
  decomposition logic itself: slab bounds, sparse ownership, restricted
  operators, exchanged plane ranges, gather.
* GPU: all ranks in one process on one device (``run_local``), real kernels
  on device windows, ghost planes copied device-to-device between steps.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_1807_03032_b200.backend.slab import (SlabRank, exchange,
                                                run_local, slab_bounds)


def _problem(so=8, n=24, nbl=4, nt=8):
    op, bufs, dt, meta = workloads.config2(so=so, n=n, nbl=nbl, nt=nt,
                                           nrec_side=12)
    H = so // 2
    rng = np.random.default_rng(7)
    inner = (slice(0, 2), slice(H, -H), slice(H, -H), slice(H, -H))
    bufs["u"].data[inner] = rng.uniform(-1, 1, bufs["u"].data[inner].shape)
    # the source sits at the x centre: at world 2 its corner planes straddle
    # the slab boundary, exercising ownership
    return op, bufs, dt, meta


def test_slab_bounds():
    assert slab_bounds(0, 9, 3, 2) == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(Exception):
        slab_bounds(0, 5, 4, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    op, bufs, dt, meta = _problem()
    nt = meta["nt"]
    rk = SlabRank(op, bufs, rank, world, nt, dry=True, dt=dt)
    # per-rank full-size host arrays; planes outside the window poisoned
    arrays = {k: v.data.copy() for k, v in rk.buffers.items()}
    for name in rk.written:
        a = arrays[name]
        a[:, :rk.xwin[0]] = np.nan
        a[:, rk.xwin[1]:] = np.nan
    local = {k: type(b)(b.name, b.dtype, arrays[k].shape, data=arrays[k])
             for k, b in rk.buffers.items()}
    x0 = rk.xwin[0]
    for t in range(nt):
        oracle.apply(rk.local_op, nt, local, dt=dt, t_m=t, t_M=t,
                     x_m=rk.a, x_M=rk.b - 1)
        for name in rk.written:
            slot = arrays[name][(t + 1) % 3]
            reqs = []
            for side, peer in ((-1, rank - 1), (+1, rank + 1)):
                if 0 <= peer < world:
                    s, r = rk.send_planes(side), rk.recv_planes(side)
                    snd = torch.from_numpy(np.ascontiguousarray(
                        slot[s.start + x0:s.stop + x0]))
                    rcv = torch.empty_like(snd)
                    reqs.append((dist.isend(snd, peer), None, None))
                    reqs.append((dist.irecv(rcv, peer), rcv, r))
            for w, rcv, r in reqs:
                w.wait()
                if rcv is not None:
                    slot[r.start + x0:r.stop + x0] = rcv.numpy()
    lo, hi = rk.owned_storage()
    res = {"u": (lo, hi, arrays["u"][:, lo:hi].copy())}
    if "rec" in local:
        res["rec"] = (rk.keep["rec"], local["rec"].data.copy())
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_bitwise():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    op, bufs, dt, meta = _problem()
    ref = oracle.apply(op, meta["nt"], bufs, dt=dt)
    u = ref["u"].copy()
    rec = np.zeros_like(ref["rec"])
    for r in range(world):
        lo, hi, part = results[r]["u"]
        u[:, lo:hi] = part
        if "rec" in results[r]:
            idx, vals = results[r]["rec"]
            rec[:, idx] = vals
    assert np.array_equal(u, ref["u"])
    assert np.array_equal(rec, ref["rec"])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_slabs_bitwise(world):
    op, bufs, dt, meta = _problem(n=40, nt=10)
    single = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
              for k, b in bufs.items()}
    op.apply(steps=meta["nt"], buffers=single, dt=dt)
    ranks = run_local(op, bufs, world, meta["nt"], dt=dt)
    out = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
           for k, b in bufs.items()}
    for rk in ranks:
        rk.gather_into(out)
    assert np.array_equal(out["u"].data, single["u"].data)
    assert np.array_equal(out["rec"].data, single["rec"].data)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_slabs_overlap_bitwise(world):
    """The overlapped step of the multi-GPU run (boundary planes + their
    sources first, ghost copies on a second stream concurrent with the
    interior part) is bitwise equal to the single-domain run."""
    op, bufs, dt, meta = _problem(n=40, nt=10)
    single = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
              for k, b in bufs.items()}
    op.apply(steps=meta["nt"], buffers=single, dt=dt)
    ranks = run_local(op, bufs, world, meta["nt"], overlap=True, dt=dt)
    assert all(rk.overlap is not None for rk in ranks)
    if world == 2:   # the source straddles the slab boundary
        assert sum(rk.overlap["n_early"] for rk in ranks) >= 1
    out = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
           for k, b in bufs.items()}
    for rk in ranks:
        rk.gather_into(out)
    assert np.array_equal(out["u"].data, single["u"].data)
    assert np.array_equal(out["rec"].data, single["rec"].data)


@pytest.mark.gpu
def test_gpu_slabs_colliding_sources_keep_point_order():
    """Two sources on the same point next to the slab boundary: the serial
    injection kernel adds them in point order, so the overlap split (which
    reorders boundary sources first) is dropped and the original order must
    come back -- bitwise equal to the single-domain run."""
    so, n, nbl, nt = 8, 40, 4, 8
    N = n + 2 * nbl
    h = 20.0
    c = h * (N - 1) / 2
    srcs = [(c - 3.1, c + 1.3, c - 2.2), (c + 4.4, c, c + 5.0),
            (c - 3.1, c + 1.3, c - 2.2)]
    op = workloads.acoustic_operator((N, N, N), h, so, srcs,
                                     [(c, c, 100.0), (c + 40.0, c, 60.0)])
    bufs = op.allocate(nt)
    bufs["m"].data[...] = np.float32(1 / 2.0 ** 2)
    bufs["damp"].data[...] = workloads.damping_profile(
        (N, N, N), nbl, so // 2).astype(np.float32)
    dt = 0.4 * h / 2.0
    w = workloads.ricker(nt, dt, 0.015)
    for p in range(3):
        bufs["src"].data[:, p] = (w * (1 + 0.37 * p)).astype(np.float32)
    single = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
              for k, b in bufs.items()}
    op.apply(steps=nt, buffers=single, dt=dt)
    ranks = run_local(op, bufs, 2, nt, overlap=True, dt=dt)
    assert all(rk.overlap is None for rk in ranks)   # serial injection
    out = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
           for k, b in bufs.items()}
    for rk in ranks:
        rk.gather_into(out)
    assert np.array_equal(out["u"].data, single["u"].data)
    assert np.array_equal(out["rec"].data, single["rec"].data)


def test_slab_rejects_stale_exchange_schedules():
    """An interpolation of u[t+1] would read a ghost plane that is only
    exchanged after the step: the decomposition refuses it."""
    import paper_1807_03032_b200.symbolic as S
    from paper_1807_03032_b200.backend.buffers import BackendError
    from paper_1807_03032_b200.backend.operator import Operator
    N, so = 24, 4
    g = S.Grid((N,) * 3, extent=(230.0,) * 3)
    u = S.FunctionDecl("u", "timefunction", g, space_order=so)
    m = S.FunctionDecl("m", "function", g, space_order=so)
    rec = S.FunctionDecl("rec", "sparsetimefunction", g, npoint=1,
                         coordinates=[(115.0, 115.0, 115.0)])
    eqs = [S.Eq(u.forward, S.solve_for(m.at * S.dt2(u) - S.laplace(u),
                                       u.forward))]
    eqs += S.interpolate(rec, u.forward)
    op = Operator(eqs, dtype="f32")
    bufs = op.allocate(4, pinned=False)
    bufs["m"].data[...] = 0.25
    with pytest.raises(BackendError, match="interpolations from t"):
        SlabRank(op, bufs, 0, 2, 4, dry=True, dt=1.0)


def _exchange_worker(rank, world, port, q):
    """The production exchange() (batched isend/irecv of the written slot's
    send planes) over gloo: every rank fills its owned planes with a
    rank-tagged pattern and checks what lands in its ghost planes."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    op, bufs, dt, meta = _problem()
    rk = SlabRank(op, bufs, rank, world, meta["nt"], dry=True,
                  overlap=True, dt=dt)
    t = 3
    ok = True
    for _, v in rk.slot_views(t):
        v.zero_()
        n = v.shape[0]
        for i in range(n):
            v[i] = 1000 * rank + i
    exchange(rk, t)
    for _, v in rk.slot_views(t):
        for side, peer in ((-1, rank - 1), (+1, rank + 1)):
            if not 0 <= peer < world:
                continue
            r = rk.recv_planes(side)
            # the neighbour's send planes, in its local window numbering
            nb = SlabRank(op, bufs, peer, world, meta["nt"], dry=True, dt=dt)
            s_ = nb.send_planes(-side)
            want = torch.stack([torch.full_like(v[0], 1000 * peer + i)
                                for i in range(s_.start, s_.stop)])
            ok &= bool(torch.equal(v[r], want))
    # the overlap split covers the slab exactly once
    ov = rk.overlap
    planes = []
    for lo, hi in ov["early"]:
        planes += list(range(lo, hi + 1))
    lo, hi = ov["interior"]
    planes += list(range(lo, hi + 1))
    ok &= sorted(planes) == list(range(rk.a, rk.b))
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_exchange_and_overlap_split():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert all(res.values()), res


@pytest.mark.gpu
@pytest.mark.parametrize("overlap", [False, True], ids=["plain", "overlap"])
@pytest.mark.parametrize("so,world", [(8, 2), (12, 3), (4, 2)])
def test_gpu_tti_slabs_bitwise(so, world, overlap):
    """TTI (config 3 shape, reduced) decomposed in x: p and r ghost planes
    exchanged every step (overlapped: boundary planes first, the interior
    while the ghosts travel); bitwise equal to the single-domain run."""
    op, bufs, dt, meta = workloads.config3(so=so, n=40, nbl=4, nt=6)
    rng = np.random.default_rng(11)
    H = so // 2
    for k in ("p", "r"):
        inner = bufs[k].data[0:2, H:-H, H:-H, H:-H]
        inner[...] = rng.uniform(-1, 1, inner.shape).astype(np.float32)
    single = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
              for k, b in bufs.items()}
    op.apply(steps=meta["nt"], buffers=single, dt=dt)
    ranks = run_local(op, bufs, world, meta["nt"], overlap=overlap, dt=dt)
    assert all((rk.overlap is not None) == overlap for rk in ranks)
    out = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
           for k, b in bufs.items()}
    for rk in ranks:
        rk.gather_into(out)
    for k in ("p", "r"):
        assert np.array_equal(out[k].data, single[k].data), k


def test_tti_weak_slab_workload_matches_config3():
    """At world 1 the weak-scaled TTI workload is config 3 itself; at world
    2 a rank's ghost planes hold its neighbour's values (repeated cube)."""
    op1, b1, dt1, _ = workloads.tti_weak_slab(1, 0, so=8, n=24, nbl=4, nt=4)
    op3, b3, dt3, _ = workloads.config3(so=8, n=24, nbl=4, nt=4)
    assert dt1 == dt3
    for k in ("m", "damp", "epsilon", "delta", "theta", "phi"):
        assert np.array_equal(b1[k].data, b3[k].data), k
    _, lo, _, _ = workloads.tti_weak_slab(2, 0, so=8, n=24, nbl=4, nt=4)
    _, hi, _, _ = workloads.tti_weak_slab(2, 1, so=8, n=24, nbl=4, nt=4)
    H, n = 4, 32
    # rank 0's upper ghost planes are rank 1's first owned planes
    assert np.array_equal(lo["theta"].data[n + H:n + 2 * H],
                          hi["theta"].data[H:2 * H])


@pytest.mark.gpu
def test_config5_field_windows_consistent():
    """The strong-scaling generator gives every rank the planes of the same
    global smoothed field (per-plane seeded noise, margins of real noise,
    edge replication only at the global ends)."""
    full = workloads._smoothed_window_gpu(7, 60, 24, 20, 0, 60, 0.0, 1.0)
    parts = [workloads._smoothed_window_gpu(7, 60, 24, 20, a, b, 0.0, 1.0)
             for a, b in ((0, 17), (17, 41), (41, 60))]
    joined = np.concatenate(parts, axis=0)
    assert joined.shape == full.shape
    assert np.abs(joined - full).max() <= 1e-6
    assert 0.0 <= full.min() and full.max() <= 1.0 and full.std() > 0.01


def test_config4_windows_tile_the_global_grid():
    """Config 4 (weak scaling): each rank's storage window is its slab plus
    so/2 ghost planes, the slabs tile the global x range, one source per
    slab lands in its own slab, and m is the config-1 two-layer model."""
    world, so, n = 3, 8, 24
    H = so // 2
    owned = []
    for rank in range(world):
        op, bufs, dt, meta = workloads.config4_slab(world, rank, so=so, n=n,
                                                    nt=4)
        a, b = meta["slab"]
        owned.append((a, b))
        assert bufs["u"].data.shape == (3, b - a + 2 * H, n + 2 * H,
                                        n + 2 * H)
        assert not bufs["damp"].data.any()
        assert set(np.unique(bufs["m"].data)) <= {np.float32(1 / 1.5 ** 2),
                                                  *bufs["m"].data[0, 0, -1:]}
        xs = bufs["src_coords"].data[:, 0] / meta["h"]
        assert a <= xs[rank] < b
    assert owned[0][0] == 0 and owned[-1][1] == n * world
    assert all(owned[i][1] == owned[i + 1][0] for i in range(world - 1))
