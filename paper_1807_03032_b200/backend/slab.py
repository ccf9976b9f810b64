"""x-slab decomposition of ``Operator.apply`` over ranks.

The loop box is split along x, the outermost storage axis, into contiguous
slabs, one per rank. A rank keeps on its device only the storage planes of
its slab plus ``halo`` ghost planes per side (``DeviceRun(xwin=...)``); at the
global ends the ghosts are the functions' own (zero) halo, exactly as on one
device. Every time step: the rank's stages run over its slab, then the
ghost planes of the just-written time slot are exchanged with the x-1 / x+1
neighbours (point-to-point; NCCL over NVLink on GPUs, gloo on CPU).

Sparse ownership (computed with the oracle's own index arithmetic, in the
global frame, so tables and weights are identical to the single-device run):

* a source point is handled by every rank whose owned planes contain one of
  its corner planes (base or base+1); corners that land in a ghost plane are
  injected too and then overwritten by the neighbour's exchanged (owned,
  injected) values -- each owned corner is injected exactly once, by its
  owner, before the exchange;
* a receiver is evaluated by the rank owning its base plane; base+1 is owned
  or a freshly exchanged ghost plane of u[t].

Per-point arithmetic is the single-device program, so the decomposed run is
bitwise identical to the single-device run (tests/test_slab.py).
"""

from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from ..symbolic.expr import Access, children_of, rebuild
from ..symbolic.grid import Equation, FunctionDecl
from ..symbolic.sparse import corner_terms
from .buffers import BackendError, DataBuffer
from .program import SparseEvaluator


def slab_bounds(lo: int, hi: int, world: int, min_planes: int
                ) -> List[Tuple[int, int]]:
    """Contiguous balanced split of loop planes [lo, hi] into ``world``
    slabs [a, b); each must hold at least ``min_planes`` planes (a ghost
    exchange only reaches the nearest neighbour)."""
    n = hi - lo + 1
    if world < 1 or n < world * max(min_planes, 1):
        raise BackendError("cannot split %d planes into %d slabs of >= %d"
                           % (n, world, min_planes))
    out, a = [], lo
    for r in range(world):
        size = n // world + (1 if r < n % world else 0)
        out.append((a, a + size))
        a += size
    return out


def _x_halo(op) -> int:
    halos = {f.halo for f in op.functions.values()
             if f.kind in ("function", "timefunction")}
    if len(halos) != 1:
        raise BackendError("slab decomposition needs one common halo, got %s"
                           % sorted(halos))
    return halos.pop()


def sparse_base_x(op, buffers: Dict[str, DataBuffer], env: dict
                  ) -> Dict[str, np.ndarray]:
    """Per sparse function: loop-x index of each point's base corner,
    evaluated with the oracle's arithmetic (floor((c - o)/h) in the operator
    dtype, reference sparse.py:19-34)."""
    out = {}
    arrays = {k: v.data for k, v in buffers.items()}
    for f in op.functions.values():
        if f.kind != "sparsetimefunction":
            continue
        base = corner_terms(f)[0][0]
        ev = SparseEvaluator(env, op.dtype, f.npoint, arrays, {},
                             f.point_dim.name, 0)
        out[f.name] = ev.index(base)
    return out


def _restrict(op, keep: Dict[str, np.ndarray]):
    """The operator's equations with every sparse function replaced by one
    over the kept points (same name, same coordinates order)."""
    # keyed by name: a cached artifact may hold other (equal) declarations
    # than the ones the operator's equations reference
    new: Dict[str, FunctionDecl] = {}
    for f in op.functions.values():
        if f.kind == "sparsetimefunction":
            idx = keep[f.name]
            coords = f.coordinate_array[idx] \
                if f.coordinate_array is not None else None
            if len(idx) == 0:
                continue
            d = FunctionDecl(f.name, f.kind, f.grid, npoint=len(idx),
                             coordinates=coords)
            new[f.name] = d
            new[f.coordinates.name] = d.coordinates

    dropped = {f.name for f in op.functions.values()
               if f.kind == "sparsetimefunction" and len(keep[f.name]) == 0}

    def tr(e):
        if isinstance(e, Access):
            d = new.get(e.func.name, e.func) \
                if e.func.kind in ("sparsetimefunction", "coordinates") \
                else e.func
            return Access(d, tuple(tr(i) for i in e.indices))
        kids = children_of(e)
        return rebuild(e, [tr(c) for c in kids]) if kids else e

    def uses_dropped(e):
        if isinstance(e, Access) and e.func.name in dropped:
            return True
        return any(uses_dropped(c) for c in children_of(e))

    eqs = []
    for eq in op.eqs:
        if uses_dropped(eq.lhs) or uses_dropped(eq.rhs):
            continue
        eqs.append(Equation(tr(eq.lhs), tr(eq.rhs), eq.region,
                            eq.is_increment))
    return eqs


class SlabRank:
    """One rank's share: restricted operator, sliced buffers, device run."""

    def __init__(self, op, buffers: Dict[str, DataBuffer], rank: int,
                 world: int, steps: int, device: Optional[int] = None,
                 dry: bool = False, overlap: bool = False, **params):
        self.op, self.rank, self.world = op, rank, world
        env = op.default_params(steps)
        env.update(params)
        self.env = env
        self.H = _x_halo(op)
        bounds = slab_bounds(int(env["x_m"]), int(env["x_M"]), world, self.H)
        self.bounds = bounds
        self.a, self.b = bounds[rank]
        base = sparse_base_x(op, buffers, env)
        self.keep: Dict[str, np.ndarray] = {}
        self.injected: List[str] = []
        base_x: Dict[str, np.ndarray] = {}
        for f in op.functions.values():
            if f.kind != "sparsetimefunction":
                continue
            bx = base[f.name]
            injected = any(eq.is_increment and any(
                isinstance(n, Access) and n.func.name == f.name
                for n in _walk(eq.rhs)) for eq in op.eqs)
            if injected:     # a corner plane (base or base+1) is owned here
                sel = (bx + 1 >= self.a) & (bx < self.b)
            else:            # the base plane is owned here
                sel = (bx >= self.a) & (bx < self.b)
                if rank == world - 1:
                    sel |= bx >= self.b
                if rank == 0:
                    sel |= bx < self.a
            self.keep[f.name] = np.nonzero(sel)[0]
            if injected:
                self.injected.append(f.name)
                base_x[f.name] = bx
        keep0 = {k: v.copy() for k, v in self.keep.items()}
        self._plan_overlap(overlap, base_x)
        # storage window: slab planes + H ghost planes per side
        self.xwin = (self.a, self.b + 2 * self.H)
        p = dict(params)
        p.update(x_m=self.a, x_M=self.b - 1)
        self._build(op, buffers, steps, device, dry, p)
        if self.overlap is not None and not dry and not self.run.can_split():
            # no split schedule (e.g. colliding sources run the serial
            # injection kernel, which adds in point order): restore the
            # original point order, so the sums are the single device's
            self.overlap = None
            if any(not np.array_equal(keep0[k], self.keep[k]) for k in keep0):
                self.run.close()
                self.keep = keep0
                self._build(op, buffers, steps, device, dry, p)
        self._check_exchange_slots()

    def _build(self, op, buffers, steps, device, dry, p):
        from .operator import Operator
        self.local_op = Operator(_restrict(op, self.keep), mode=op.mode,
                                 dtype=op.dtype)
        self.buffers = self._local_buffers(buffers)
        self.run = self.local_op.prepare(steps, self.buffers, device=device,
                                         dry=dry, xwin=self.xwin, **p)
        self.written = [n for n in dict.fromkeys(self.run.written)
                        if op.functions[n].kind == "timefunction"]

    def _check_exchange_slots(self):
        """The exchange after step t ships the time slot written at t
        (t + 1); that is complete only if every dense stage writes t + 1,
        injections add into t + 1 (before the exchange) and interpolations
        read t (exchanged one step earlier). Other schedules would read or
        leave stale ghost planes: rejected."""
        plan = self.run.plan
        for i in range(plan.ndense):
            d = plan.dense[i]
            if d.fast_kind != 3 and d.target.tshift != 1:
                raise BackendError("slab decomposition needs dense updates of "
                                   "t+1 (stage %d writes t%+d)"
                                   % (i, d.target.tshift))
        for i in range(plan.nsparse):
            sp = plan.sparse[i]
            want = 1 if sp.kind == 0 else 0
            if sp.field_tshift != want:
                raise BackendError(
                    "slab decomposition needs injections into t+1 and "
                    "interpolations from t (sparse stage %d %s t%+d)"
                    % (i, "injects into" if sp.kind == 0 else "reads",
                       sp.field_tshift))

    def _plan_overlap(self, overlap: bool, base_x: Dict[str, np.ndarray]):
        """Split of a time step for overlapping the ghost exchange with the
        interior: the planes a neighbour needs (H per side) plus one are
        computed first, together with the sources having a corner in them
        (kept first in the point order, so they are points [0, n_early));
        the exchange then runs while the interior planes and the remaining
        sources are computed. Per-point arithmetic is unchanged."""
        self.overlap = None
        # overlap == "force": plan the split even without neighbours (one
        # GPU measuring the split schedule's own cost; nothing is exchanged)
        force = overlap == "force"
        if not overlap or (self.world == 1 and not force) or \
                len(self.injected) > 1:
            return
        H, a, b = self.H, self.a, self.b
        lo_side = self.rank > 0 or force
        hi_side = self.rank < self.world - 1 or force
        e_lo = (a, a + H) if lo_side else None
        e_hi = (b - H - 1, b - 1) if hi_side else None
        i_lo = a + (H + 1 if lo_side else 0)
        i_hi = b - 1 - (H + 1 if hi_side else 0)
        whole = i_hi < i_lo or (e_lo and e_hi and e_lo[1] >= e_hi[0])
        if whole:                        # thin slab: everything is early
            e_lo, e_hi, i_lo, i_hi = (a, b - 1), None, 0, -1
        n_early = 0
        for name in self.injected:
            idx = self.keep[name]
            bx = base_x[name][idx]
            early = np.zeros(len(idx), bool)
            if lo_side:
                early |= (bx + 1 >= a) & (bx <= a + H - 1)
            if hi_side:
                early |= (bx + 1 >= b - H) & (bx <= b - 1)
            if whole:
                early[:] = True
            order = np.concatenate([np.nonzero(early)[0],
                                    np.nonzero(~early)[0]])
            self.keep[name] = idx[order]
            n_early = int(early.sum())
        self.overlap = {"early": [r for r in (e_lo, e_hi) if r],
                        "interior": (i_lo, i_hi), "n_early": n_early}

    def _local_buffers(self, buffers):
        out = {}
        for name, f in self.local_op.functions.items():
            src = buffers[name]
            if f.kind == "sparsetimefunction":
                data = np.ascontiguousarray(src.data[:, self.keep[name]])
            elif f.kind == "coordinates":
                owner = name[:-len("_coords")]
                data = np.ascontiguousarray(src.data[self.keep[owner]])
            else:
                data = src.data            # windowed at upload
            out[name] = DataBuffer(name, src.dtype, data.shape, data=data)
        return out

    # -- ghost planes (local storage x indices of the device window) --------

    def send_planes(self, side: int) -> slice:
        """Owned planes that the neighbour on ``side`` (-1 / +1) needs."""
        H = self.H
        if side < 0:
            return slice(H, 2 * H)                   # loop [a, a+H)
        n = self.b - self.a
        return slice(n, n + H)                       # loop [b-H, b)

    def recv_planes(self, side: int) -> slice:
        H = self.H
        if side < 0:
            return slice(0, H)                       # loop [a-H, a)
        n = self.b - self.a
        return slice(n + H, n + 2 * H)               # loop [b, b+H)

    def slot_views(self, t: int):
        """(name, tensor of the time slot written at step t) per written
        time function."""
        out = []
        for name in self.written:
            f = self.op.functions[name]
            slot = (t + 1) % f.time_dim.modulo
            out.append((name, self.run.dev[name][slot]))
        return out

    def owned_storage(self) -> Tuple[int, int]:
        """Global storage x planes this rank owns (plus the outer halo at
        the global ends)."""
        H = self.H
        lo = self.a + H if self.rank else 0
        hi = self.b + H if self.rank < self.world - 1 else self.b + 2 * H
        return lo, hi

    def gather_into(self, buffers: Dict[str, DataBuffer]):
        """Write this rank's owned results into (global) host buffers: dense
        planes in place (the rank's dense buffers alias the global arrays or
        are windows of them), sparse columns by point index."""
        self.run.download(xrange=self.owned_storage())
        if any(self.buffers[n].data is not buffers[n].data
               for n in self.written):
            lo, hi = self.owned_storage()
            for name in self.written:
                src = self.buffers[name].data
                off = 0 if src.shape[1] == buffers[name].data.shape[1] \
                    else self.xwin[0]
                buffers[name].data[:, lo:hi] = src[:, lo - off:hi - off]
        for name, f in self.local_op.functions.items():
            if f.kind == "sparsetimefunction" and name in self.run.written:
                buffers[name].data[:, self.keep[name]] = \
                    self.buffers[name].data


def _walk(e):
    yield e
    for c in children_of(e):
        yield from _walk(c)


def run_local(op, buffers: Dict[str, DataBuffer], world: int, steps: int,
              device: Optional[int] = None, overlap: bool = False,
              **params) -> List[SlabRank]:
    """All ranks of a decomposition in ONE process on one device, stepped
    in turn with device-to-device ghost copies between steps: validates the
    decomposition bit for bit on a single GPU without ranks that wait on
    each other. ``overlap``: the split step of the multi-GPU run (boundary
    part, ghost copies on a second stream concurrent with the interior
    part, join before the next step)."""
    import torch
    ranks = [SlabRank(op, buffers, r, world, steps, device=device,
                      overlap=overlap, **params) for r in range(world)]
    t_m, t_M = int(ranks[0].env["t_m"]), int(ranks[0].env["t_M"])

    def copies(t):
        for r in range(world - 1):
            lo, hi = ranks[r], ranks[r + 1]
            for (_, vl), (_, vh) in zip(lo.slot_views(t), hi.slot_views(t)):
                vh[hi.recv_planes(-1)].copy_(vl[lo.send_planes(+1)])
                vl[lo.recv_planes(+1)].copy_(vh[hi.send_planes(-1)])

    split = overlap and all(rk.overlap is not None for rk in ranks)
    comp = torch.cuda.current_stream()
    comm = torch.cuda.Stream()
    for t in range(t_m, t_M + 1):
        if not split:
            for rk in ranks:
                rk.run.step(t)
            copies(t)
            continue
        for rk in ranks:
            step_boundary(rk, t)
        comm.wait_stream(comp)
        with torch.cuda.stream(comm):
            copies(t)
        for rk in ranks:
            step_interior(rk, t)
        comp.wait_stream(comm)
    torch.cuda.synchronize()
    return ranks


def run_distributed(op, buffers: Dict[str, DataBuffer], steps: int,
                    device: Optional[int] = None, **params) -> SlabRank:
    """This process's rank of a torch.distributed run (NCCL on GPUs):
    per step, launch the slab's stages then exchange ghost planes with
    batched isend/irecv on the current stream -- no host synchronisation."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    rk = SlabRank(op, buffers, rank, world, steps, device=device,
                  overlap=True, **params)
    step_loop(rk)
    torch.cuda.synchronize()
    return rk


def exchange(rk: SlabRank, t: int) -> None:
    """Ghost-plane exchange after step t: the slot written at t goes to the
    x-1 / x+1 neighbours with batched isend/irecv (NCCL stream ordered
    after the step's kernels; the current stream waits for completion)."""
    import torch.distributed as dist
    cache = rk.__dict__.setdefault("_xchg", {})
    key = tuple((name, v.data_ptr()) for name, v in rk.slot_views(t))
    ops = cache.get(key)
    if ops is None:                      # one op list per time slot
        ops = []
        for _, v in rk.slot_views(t):
            if rk.rank > 0:
                ops.append(dist.P2POp(dist.isend, v[rk.send_planes(-1)],
                                      rk.rank - 1))
                ops.append(dist.P2POp(dist.irecv, v[rk.recv_planes(-1)],
                                      rk.rank - 1))
            if rk.rank < rk.world - 1:
                ops.append(dist.P2POp(dist.isend, v[rk.send_planes(+1)],
                                      rk.rank + 1))
                ops.append(dist.P2POp(dist.irecv, v[rk.recv_planes(+1)],
                                      rk.rank + 1))
        cache[key] = ops
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def step_boundary(rk: SlabRank, t: int) -> None:
    """First part of an overlapped step t (current stream): the planes the
    neighbours need (+1) and the sources touching them."""
    run, ov = rk.run, rk.overlap
    for lo, hi in ov["early"]:
        run.step_part(t, run.DENSE, x_lo=lo, x_hi=hi)
    if ov["n_early"]:
        run.step_part(t, run.INJECT, p_lo=0, p_hi=ov["n_early"])


def step_interior(rk: SlabRank, t: int) -> None:
    """Second part of an overlapped step t: interior planes, remaining
    sources, receivers (which read u[t], exchanged at step t - 1)."""
    run, ov = rk.run, rk.overlap
    lo, hi = ov["interior"]
    if hi >= lo:
        run.step_part(t, run.DENSE, x_lo=lo, x_hi=hi)
    run.step_part(t, run.INJECT, p_lo=ov["n_early"])
    run.step_part(t, run.INTERP)


def step_once(rk: SlabRank, t: int) -> None:
    """Time step t of this rank: slab stages and the ghost exchange. With
    ``rk.overlap`` the exchange runs on a communication stream while the
    interior of step t is computed; step t + 1 waits for it."""
    import torch
    if rk.overlap is None:
        rk.run.step(t)
        if rk.world > 1:
            exchange(rk, t)
        return
    if rk.world == 1:                    # forced split, nothing to exchange
        step_boundary(rk, t)
        step_interior(rk, t)
        return
    comp = torch.cuda.current_stream()
    comm = getattr(rk, "_comm", None)
    if comm is None:
        comm = rk._comm = torch.cuda.Stream()
    step_boundary(rk, t)
    comm.wait_stream(comp)
    with torch.cuda.stream(comm):
        exchange(rk, t)
    step_interior(rk, t)
    comp.wait_stream(comm)


def step_loop(rk: SlabRank) -> None:
    """t_m..t_M of this rank: the library's data plane when attached
    (attach_native: one CUDA graph per rank with NCCL send/recv inside),
    else the host-driven loop of step_once."""
    if getattr(rk, "xspec", None) is not None:
        import torch
        prep = rk.run.prepared()
        prep.multi_run(rk.comm, rk.xspec,
                       torch.cuda.current_stream(rk.run.device).cuda_stream)
        return
    for t in range(int(rk.env["t_m"]), int(rk.env["t_M"]) + 1):
        step_once(rk, t)


def exchange_spec(rk: SlabRank, lo_peer: Optional[int] = None,
                  hi_peer: Optional[int] = None):
    """sc_exchange of a rank: the written time functions, its neighbours and
    the overlap split in the run's local loop coordinates."""
    from . import runtime as rt
    x = rt.ScExchange()
    if len(rk.written) > 4:
        raise BackendError("at most 4 exchanged time functions")
    x.nfields = len(rk.written)
    for i, n in enumerate(rk.written):
        x.field[i] = rk.run.field_ids[n]
    x.lo_peer = (rk.rank - 1 if rk.rank > 0 else -1) if lo_peer is None \
        else lo_peer
    x.hi_peer = (rk.rank + 1 if rk.rank < rk.world - 1 else -1) \
        if hi_peer is None else hi_peer
    x.halo, x.slab = rk.H, rk.b - rk.a
    ov = rk.overlap
    if ov is not None:
        sh = rk.run.xshift
        x.overlap = 1
        x.nearly = len(ov["early"])
        for k, (lo, hi) in enumerate(ov["early"]):
            x.early[k][0], x.early[k][1] = lo - sh, hi - sh
        lo, hi = ov["interior"]
        x.interior[0], x.interior[1] = (lo - sh, hi - sh) if hi >= lo \
            else (0, -1)
        x.n_early_points = ov["n_early"]
    return x


def make_comm(rank: int, world: int):
    """The library's NCCL communicator (sc_multi_init); the unique id goes
    from rank 0 to the others over the torch.distributed process group
    (plumbing only: no data-path collective)."""
    import torch
    import torch.distributed as dist
    from . import runtime as rt
    uid = rt.multi_unique_id() if rank == 0 else bytes(128)
    if world > 1:
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().tolist())
    return rt.MultiComm(uid, rank, world)


def attach_native(rk: SlabRank, comm=None) -> SlabRank:
    """Run this rank's t loop through the library (sc_multi_run): ``comm``
    from make_comm, or None when the rank has no neighbours."""
    rk.comm = comm
    rk.xspec = exchange_spec(rk)
    if (rk.xspec.lo_peer >= 0 or rk.xspec.hi_peer >= 0) and comm is None:
        raise BackendError("a rank with neighbours needs a communicator")
    return rk
