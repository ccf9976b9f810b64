"""``Operator``: the drop-in for the reference's compile-and-apply driver.

Same constructor and runtime surface as the reference
(pkg/src/stencilc/backend/operator.py:138-253):

* ``Operator(eqs, mode="advanced", block=None, dtype="f64", subs=None,
  name="kernel")`` lowers, clusters and optimizes the equations (restated
  passes, identical trees) and caches the artifact by content hash
  (operator.py:67-88, 141-158);
* ``allocate(steps)`` -> zeroed ``DataBuffer`` per function, coordinates
  filled (operator.py:181-195);
* ``default_params(steps)`` -> spacing/origin bindings and loop bounds capped
  by the data spaces (operator.py:197-233);
* ``apply(steps=1, buffers=None, workers=1, **params) -> (buffers, report)``
  runs the whole time loop on the GPU (operator.py:235-244), mutating the
  caller's numpy buffers in place; ``report`` maps section names to
  ``{"time", "points"}`` (interpreter.py:117-124).

Execution never falls back to the CPU: unsupported equations or a missing
GPU/library raise ``BackendError``.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from ..symbolic.expr import (Access, Add, Constant, Expr, Mul, Pow, Symbol,
                             children_of, free_symbols)
from ..symbolic.grid import Equation, FunctionDecl, Grid
from . import dse as _dse
from . import runtime as rt
from .buffers import DTYPES, BackendError, BoundsError, DataBuffer
from .fastpath import match_acoustic
from .recognize import match_tti
from .lowering import (OPAQUE, LoweredEq, _deep_accesses, access_offsets,
                       collect_functions,
                       lower, shift_of)
from .program import (DenseProgram, SparseEvaluator, _Vec, compile_dense,
                      program_trace)

PASS_WORK = 0
_CACHE: Dict[str, "Artifact"] = {}


def clear_cache():
    _CACHE.clear()


@dataclass
class Artifact:
    key: str
    lowered: List[LoweredEq]
    clusters: List[_dse.Cluster]
    functions: Dict[str, FunctionDecl]
    grid: Grid
    sections: List[str]
    pass_times: Dict[str, float] = field(default_factory=dict)


def _decl_signature(f: FunctionDecl) -> tuple:
    g, td = f.grid, f.time_dim
    arr = getattr(f, "coordinate_array", None)
    coords = hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest() \
        if arr is not None else None
    return (f.name, f.kind, g.shape, g.extent, g.origin, f.space_order,
            f.time_order, f.save, f.npoint, f.padding,
            (td.kind, td.factor, td.modulo) if td else None, coords,
            getattr(f, "nt", None))


def _content_key(eqs, mode, block, dtype, subs) -> str:
    h = hashlib.sha256()
    decls: Dict[str, FunctionDecl] = {}
    for eq in eqs:
        h.update(repr((eq.lhs, eq.rhs, eq.region, eq.is_increment)).encode())
        h.update(b"\0")
        stack = [eq.lhs, eq.rhs]
        while stack:
            e = stack.pop()
            if isinstance(e, Access) and e.func.kind != "temp":
                decls.setdefault(e.func.name, e.func)
            stack.extend(children_of(e))
    for n in sorted(decls):
        h.update(repr(_decl_signature(decls[n])).encode())
        h.update(b"\0")
    bpart = tuple(sorted(block.items())) if isinstance(block, dict) else block
    spart = tuple(sorted((repr(k), repr(v)) for k, v in (subs or {}).items()))
    h.update(repr((mode, bpart, dtype, spart)).encode())
    return h.hexdigest()


#: internal mode of ``Operator.reference``: the lowered equations exactly as
#: written (no clustering, no DSE, no family kernels)
UNOPTIMIZED = "unoptimized"


def _unoptimized_clusters(lowered) -> List[_dse.Cluster]:
    """reference_run's schedule (reference interpreter.py:493-549): one loop
    nest per lowered equation in program order; every equation with a time
    dimension runs inside the single outer time loop (time first)."""
    out = []
    for eq in lowered:
        dims = tuple(eq.dims)
        tdims = [d for d in dims if d.is_time]
        if tdims:
            dims = tuple(tdims) + tuple(d for d in dims if not d.is_time)
        out.append(_dse.Cluster([eq], dims, guards=eq.guards))
    return out


def _compile(eqs, mode, dtype, subs, fuse=True) -> Artifact:
    global PASS_WORK
    times = {}
    t0 = time.perf_counter()
    lowered = [lower(e, subs) for e in eqs]
    times["lowering"] = time.perf_counter() - t0
    functions = collect_functions(lowered)
    if not functions:
        raise BackendError("operator touches no declared function")
    grid = next(iter(functions.values())).grid
    if mode == UNOPTIMIZED:
        clusters = _unoptimized_clusters(lowered)
        PASS_WORK += 1
        statics = [c for c in clusters if not any(d.is_time for d in c.dims)]
        nsec = len(statics) + len(_device_phases(clusters))
        return Artifact(_content_key(eqs, mode, None, dtype, subs), lowered,
                        clusters, functions, grid,
                        ["section%d" % i for i in range(nsec)], times)
    # recognised families with a dedicated (non-exact-order) kernel skip the
    # DSE: TTI's optimized tree costs the reference 10-941 s to build
    tti = match_tti(list(eqs)) if fuse and not subs else None
    rest = list(range(len(lowered)))
    fused = None
    if tti is not None:
        i, j, roles = tti
        rest = [k for k in rest if k not in (i, j)]
        fused = _dse.Cluster([lowered[i], lowered[j]], lowered[i].dims,
                             fused=("tti", roles))
    t0 = time.perf_counter()
    clusters = _dse.clusterize([lowered[k] for k in rest])
    times["clustering"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    clusters = _dse.run_dse(clusters, mode, grid)
    times["dse"] = time.perf_counter() - t0
    if fused is not None:
        first_timed = next((k for k, c in enumerate(clusters)
                            if any(d.is_time for d in c.dims)), len(clusters))
        clusters.insert(first_timed, fused)
    PASS_WORK += 3
    # top-level loop nests, one section each: hoisted producers, then the
    # time loop (reference operator.py:124-125)
    statics = [c for c in clusters if not any(d.is_time for d in c.dims)]
    nsec = len(statics) + len(_device_phases(clusters))
    sections = ["section%d" % i for i in range(nsec)]
    return Artifact(_content_key(eqs, mode, None, dtype, subs), lowered,
                    clusters, functions, grid, sections, times)


def _time_outer(c) -> bool:
    return bool(c.dims) and c.dims[0].is_time


def _device_phases(clusters) -> List[list]:
    """Top-level loop nests after the hoisted producers, in program order
    (reference iet.py build_iet: consecutive clusters share the outer t
    loop; a cluster whose iteration space has time inside the space dims,
    e.g. ``img[x, y] += us[t/f, x, y] * u[t, x, y]``, is a nest of its own
    run after the preceding t loop has finished)."""
    phases: List[list] = []
    for c in clusters:
        if not any(d.is_time for d in c.dims):
            continue
        if _time_outer(c) and phases and _time_outer(phases[-1][-1]):
            phases[-1].append(c)
        else:
            phases.append([c])
    return phases


class Operator:
    """A compiled, cached stencil operator executed on B200 GPUs."""

    def __init__(self, eqs: Sequence[Equation], mode: str = "advanced",
                 block: Optional[Dict[str, int]] = None, dtype: str = "f64",
                 subs: Optional[dict] = None, name: str = "kernel",
                 fuse: bool = True):
        """``fuse=False`` disables the recognised-family kernels whose
        arithmetic order differs from the oracle's (TTI); every statement
        then goes through the exact path."""
        if not eqs:
            raise BackendError("operator needs at least one equation")
        if dtype not in DTYPES:
            raise BackendError("bad dtype %r" % dtype)
        if mode not in _dse.MODES and mode != UNOPTIMIZED:
            raise ValueError("unknown optimization mode %r" % mode)
        self.eqs = list(eqs)
        self.mode = mode
        self.block = dict(block) if block else None
        self.dtype = dtype
        self.subs = subs
        self.name = name
        key = _content_key(self.eqs, mode, None, dtype, subs) + \
            ("" if fuse else ":nofuse")
        art = _CACHE.get(key)
        self.cache_hit = art is not None
        if art is None:
            art = _compile(self.eqs, mode, dtype, subs, fuse)
            _CACHE[key] = art
        self.artifact = art

    @property
    def grid(self) -> Grid:
        return self.artifact.grid

    @property
    def functions(self) -> Dict[str, FunctionDecl]:
        return self.artifact.functions

    @property
    def clusters(self):
        return self.artifact.clusters

    @property
    def iet(self) -> "IetNode":
        """Loop-nest tree of the compiled operator (reference
        operator.py:160-162 exposes its IET): a root ``Block`` whose children
        are the sections in execution order, each holding its loop nest and
        the clusters (statements) it runs. Built on access; see ``dump_iet``."""
        return build_iet(self)

    def dump_iet(self) -> str:
        return self.iet.dump()

    @property
    def source(self) -> str:
        """What runs on the device (reference operator.py:164-166 returns its
        emitted C): per section, the kernel family chosen for every cluster
        (fused acoustic, fused TTI, NVRTC-generated program kernel, sparse
        inject/interpolate) and the statements it executes, followed by the
        straight-line programs the generic kernels compile."""
        return device_source(self)

    # -- buffers and bounds ------------------------------------------------------

    def allocate(self, steps: int, pinned: Optional[bool] = None
                 ) -> Dict[str, DataBuffer]:
        """Zeroed buffers (reference operator.py:181-195). On a GPU host the
        arrays live in page-locked memory so apply()'s host<->device copies
        run as DMA; they are ordinary numpy arrays to the caller."""
        if pinned is None:
            pinned = _cuda_available()
        for f in self.functions.values():
            # Devito-style SparseTimeFunction(nt=...): the reference sizes
            # sparse time axes by ``steps`` (operator.py:185-190), so the two
            # must agree
            nt = getattr(f, "nt", None)
            if f.kind == "sparsetimefunction" and nt is not None and \
                    int(nt) != int(steps):
                raise BackendError("%s declares nt=%d but the operator "
                                   "allocates %d time steps" %
                                   (f.name, int(nt), int(steps)))
        bufs: Dict[str, DataBuffer] = {}
        for f in self.functions.values():
            nt = steps if f.kind == "sparsetimefunction" else None
            ext = f.storage_extents(nt)
            data = _pinned_zeros(ext, self.dtype) if pinned and \
                f.kind != "coordinates" else None
            bufs[f.name] = DataBuffer(f.name, self.dtype, ext, data=data)
        for f in self.functions.values():
            if f.kind == "sparsetimefunction" and \
                    f.coordinate_array is not None and \
                    f.coordinates.name in bufs:
                bufs[f.coordinates.name].data[:] = f.coordinate_array
        return bufs

    def default_params(self, steps: int) -> dict:
        env = dict(self.grid.symbol_values())
        g = self.grid
        for i, d in enumerate(g.dimensions):
            env[d.name + "_m"] = 0
            env[d.name + "_M"] = g.shape[i] - 1
        env["t_m"] = 0
        env["t_M"] = steps - 1
        for f in self.functions.values():
            if f.kind == "sparsetimefunction":
                env[f.point_dim.name + "_m"] = 0
                env[f.point_dim.name + "_M"] = f.npoint - 1
        for eq in self.artifact.lowered:
            for decl, slot in eq.dspace.values():
                ext = decl.storage_extents(
                    steps if decl.kind == "sparsetimefunction" else None)
                for pos, (lo, hi) in slot.items():
                    d = decl.dims[pos]
                    if d.kind == "stepping":
                        continue
                    if d.kind == "conditional":
                        cap, name = d.factor * ext[pos] - 1, d.root.name
                    else:
                        cap = ext[pos] - 1 - shift_of(decl, d) - hi
                        name = d.root.name
                    if name + "_M" in env:
                        env[name + "_M"] = min(env[name + "_M"], cap)
        return env

    # -- execution ------------------------------------------------------------------

    def _steps(self, steps: Optional[int], params: dict) -> int:
        """``steps`` as given, else (Devito facade) ``time_M - time_m + 1``,
        else a declared sparse ``nt``, else 1 (the reference's default)."""
        if steps is not None:
            return int(steps)
        tM = params.get("time_M", params.get("t_M"))
        if tM is not None:
            return int(tM) - int(params.get("time_m", params.get("t_m", 0))) + 1
        nts = {int(f.nt) for f in self.functions.values()
               if getattr(f, "nt", None) is not None}
        return nts.pop() if len(nts) == 1 else 1

    def prepare(self, steps: Optional[int] = None,
                buffers: Optional[Dict[str, DataBuffer]] = None,
                device: Optional[int] = None, dry: bool = False,
                xwin: Optional[Tuple[int, int]] = None,
                **params) -> "DeviceRun":
        """Validate, compile the per-step programs and move every buffer to
        the GPU; ``DeviceRun.run()`` then executes the time loop."""
        steps = self._steps(steps, params)
        if buffers is None:
            buffers = self.allocate(steps)
        env = self.default_params(steps)
        if "time_M" in params:          # Devito spelling (facade)
            params.setdefault("t_M", params.pop("time_M"))
        if "time_m" in params:
            params.setdefault("t_m", params.pop("time_m"))
        env.update(params)
        return DeviceRun(self, buffers, env, device, dry, xwin)

    def apply(self, steps: Optional[int] = None,
              buffers: Optional[Dict[str, DataBuffer]] = None,
              workers: int = 1, **params
              ) -> Tuple[Dict[str, DataBuffer], dict]:
        """Run t_m..t_M on the GPU; results land in ``buffers`` in place.
        ``workers`` is accepted for signature compatibility (results never
        depend on it, as in the reference: test_backend.py:166-171)."""
        steps = self._steps(steps, params)
        if buffers is None:
            buffers = self.allocate(steps)
        run = _reuse_run(self, steps, buffers, params)
        if run is None:
            run = self.prepare(steps, buffers, **params)
        ok = False
        try:
            # download() follows at once: rows of interpolated functions may
            # leave while the loop still runs
            report = run.run(early_download=True)
            run.download()
            ok = True
        finally:
            _keep_run(self, steps, params, run if ok else None)
            if not ok:
                run.close()
        return buffers, report

    def release(self) -> None:
        """Free the device state a previous apply kept for reuse."""
        if _RUN_CACHE["op"] is self:
            _drop_cached_run()

    def reference(self, steps: Optional[int] = None,
                  buffers: Optional[Dict[str, DataBuffer]] = None,
                  **params) -> Dict[str, DataBuffer]:
        """The reference's oracle-of-the-oracle (operator.py:246-253 ->
        interpreter.py:493-549): the *unoptimized* lowered equations -- no
        CSE, no factorization, no hoisting, no family kernels -- each its own
        loop nest in program order inside one time loop, executed on the GPU
        by the exact program kernels (same operations in the same order as
        the reference's whole-array sweeps and per-point evaluation)."""
        op = Operator(self.eqs, mode=UNOPTIMIZED, dtype=self.dtype,
                      subs=self.subs, name=self.name)
        bufs, _ = op.apply(steps, buffers, **params)
        return bufs


# ---------------------------------------------------------------------------
# Prepared-run reuse across applies.
#
# A prepare builds the host tables, allocates the device buffers, compiles
# the per-stage programs and captures the time loop as a CUDA graph; an
# apply that repeats the same operator, buffer shapes and parameters only
# needs the host -> device copies, the graph launch and the downloads. One
# run is kept process-wide (the device buffers of one problem); it is reused
# only when every host value that fed a per-point table is bitwise unchanged
# and the fused kernels' per-apply preconditions still hold on the new data
# (sc_revalidate). SC_NO_RUN_CACHE=1 disables reuse.

_RUN_CACHE: dict = {"op": None, "key": None, "run": None}


def _run_key(op, steps, params):
    env = op.default_params(steps)
    p = dict(params)
    if "time_M" in p:
        p.setdefault("t_M", p.pop("time_M"))
    if "time_m" in p:
        p.setdefault("t_m", p.pop("time_m"))
    env.update(p)
    return (op.artifact.key, int(steps),
            tuple(sorted((k, repr(v)) for k, v in env.items())))


def _drop_cached_run():
    run = _RUN_CACHE["run"]
    _RUN_CACHE.update(op=None, key=None, run=None)
    if run is not None:
        run.close()


def _reuse_run(op, steps, buffers, params):
    import os
    if _RUN_CACHE["run"] is not None and _RUN_CACHE["op"] is not op:
        # another operator's device state: free it before this one allocates
        _drop_cached_run()
    if os.environ.get("SC_NO_RUN_CACHE") or _RUN_CACHE["op"] is not op:
        return None
    run = _RUN_CACHE["run"]
    try:
        key = _run_key(op, steps, params)
    except Exception:
        return None
    sig = tuple(sorted((k, tuple(b.data.shape), str(b.data.dtype))
                       for k, b in buffers.items() if k in op.functions))
    if key != _RUN_CACHE["key"] or sig != run.signature() or \
            any(b.data.dtype != run.np_t for k, b in buffers.items()
                if k in op.functions) or \
            not run.inputs_unchanged(buffers):
        _drop_cached_run()
        return None
    run.rebind(buffers)
    if not run.revalidate():
        _drop_cached_run()
        return None
    return run


def _keep_run(op, steps, params, run):
    import os
    if _RUN_CACHE["run"] is not None and _RUN_CACHE["run"] is not run:
        _drop_cached_run()
    if run is None or os.environ.get("SC_NO_RUN_CACHE") or \
            run.xwin is not None or run.post_plans:
        if run is not None and _RUN_CACHE["run"] is run:
            _RUN_CACHE.update(op=None, key=None, run=None)
        if run is not None:
            run.close()
        return
    _RUN_CACHE.update(op=op, key=_run_key(op, steps, params), run=run)


def _check_interchange(c):
    """A time-inner nest (x, y, t) runs on the device as t-outer sweeps;
    that is the same computation when every statement is pointwise in the
    function it writes (reads of it at the written point only) and writes
    no time-indexed data."""
    from .lowering import access_offsets, _deep_accesses
    for eq in c.eqs:
        f = eq.lhs.func
        if f.kind != "function":
            raise BackendError("time-inner loop nest writing %s is not "
                               "supported by the B200 backend" % f.name)
        own = [k for _, _, _, k in access_offsets(eq.lhs)]
        for acc in _deep_accesses(eq.rhs):
            if acc.func is f and [k for _, _, _, k in access_offsets(acc)] != own:
                raise BackendError("time-inner loop nest reads %s off the "
                                   "written point" % f.name)


def _guard(c) -> int:
    """Step divisor of a guarded cluster (t % f == 0), 0 if unguarded."""
    if not c.guards:
        return 0
    if len({f for _, f in c.guards}) > 1:
        raise BackendError("several sub-sampling factors in one statement")
    return c.guards[0][1]


FAC_SPARSE, FAC_TABLE, FAC_CONST, FAC_FIELD = 0, 1, 2, 3


def _torch():
    try:
        import torch
    except ImportError as e:  # pragma: no cover
        raise BackendError("torch is required for device buffers: %s" % e)
    if not torch.cuda.is_available():
        raise BackendError("no CUDA device available: the B200 backend has "
                           "no CPU fallback")
    return torch


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _pinned_zeros(shape, dtype):
    """numpy view of a zeroed page-locked torch tensor (kept alive by the
    array's base)."""
    import torch
    tdt = torch.float32 if dtype == "f32" else torch.float64
    t = torch.zeros(tuple(shape), dtype=tdt, pin_memory=True)
    return t.numpy()


def _ld_range(ld, lo, hi):
    return [(lo[d] + ld.offs[d], hi[d] + ld.offs[d]) for d in range(len(lo))]


class DeviceRun:
    """One apply() worth of state: device buffers, compiled stage programs
    and the C plan."""

    def __init__(self, op: Operator, buffers: Dict[str, DataBuffer],
                 env: dict, device: Optional[int], dry: bool = False,
                 xwin: Optional[Tuple[int, int]] = None):
        """``xwin=(s0, s1)``: only storage x planes [s0, s1) of the dense
        functions live on the device (an x-slab with its ghost planes,
        backend/slab.py); loop bounds and sparse indices stay global and
        are shifted into the window."""
        self.op = op
        self.xwin = xwin
        self.buffers = buffers
        self.env = env
        self.dtype = op.dtype
        self.np_t = DTYPES[op.dtype]
        self.grid = op.grid
        self.report: dict = {}
        self._keep: list = []           # host arrays referenced by the plan
        self.host_sections: List[Tuple[str, float, int]] = []
        # host-side gathers that fed per-point tables (re-checked before a
        # cached run is reused, Operator.apply)
        self.reads: list = []
        self._validate_buffers()
        self._host_prework()
        # dry=True builds the plan over host tensors (host-logic tests on
        # machines without a GPU); such a plan is never executed
        self.dry = dry
        if dry:
            import torch
            self._torch = torch
            self.device = "cpu"
        else:
            self._torch = _torch()
            self.device = self._torch.cuda.current_device() if device is None \
                else device
        self._upload()
        self._build_plan()
        self.dead = self._dead_on_entry()

    # -- host-side checks and time-invariant tables -------------------------------

    def _validate_buffers(self):
        for f in self.op.functions.values():
            if f.name not in self.buffers:
                raise BackendError("no buffer for %s" % f.name)
            b = self.buffers[f.name]
            if b.data.dtype != self.np_t:
                raise BackendError("buffer %s has dtype %s, operator is %s"
                                   % (f.name, b.data.dtype, self.dtype))
        for k in ("t_m", "t_M"):
            if k not in self.env:
                raise BackendError("unbound %s" % k)
        self.t_m, self.t_M = int(self.env["t_m"]), int(self.env["t_M"])

    def _arrays(self) -> Dict[str, np.ndarray]:
        return {k: v.data for k, v in self.buffers.items()}

    def _host_prework(self):
        """Time-invariant producer clusters (hoisted sparse weight tables,
        reference dse.py:562-607): evaluated once per apply with the
        oracle's float32 semantics, exposed in ``buffers`` like the
        reference's temps (interpreter.py:438-442)."""
        clusters = self.op.clusters
        self.static = [c for c in clusters
                       if not any(d.is_time for d in c.dims)]
        phases = _device_phases(clusters)
        if any(_time_outer(p[0]) for p in phases[1:]):
            raise BackendError("a time loop after a time-inner loop nest is "
                               "not supported by the B200 backend")
        self.timed = phases[0] if phases and _time_outer(phases[0][0]) else []
        self.post = [p[0] for p in phases if not _time_outer(p[0])]
        for c in self.post:
            _check_interchange(c)
        self.tables: Dict[str, np.ndarray] = {}
        for c in self.static:
            t0 = time.perf_counter()
            if any(d.kind == "space" for d in c.dims):
                raise BackendError("time-invariant dense clusters are not "
                                   "supported by the B200 backend")
            pdim = [d for d in c.dims if d.kind == "sparse"][0]
            lo, hi = self._prange(pdim)
            n = hi - lo + 1
            ev = SparseEvaluator(self.env, self.dtype, n, self._arrays(), {},
                                 pdim.name, lo, reads=self.reads)
            for eq in c.eqs:
                f = eq.lhs.func
                v = ev.ev(eq.rhs)
                if f.kind == "temp" and not eq.lhs.indices:
                    ev.temps[f.name] = v
                    continue
                if f.kind != "temp":
                    raise BackendError("hoisted cluster writes %s" % f.name)
                arr = np.zeros(n, self.np_t)
                arr[:] = np.broadcast_to(np.asarray(v.v).astype(self.np_t),
                                         (n,))
                self.tables[f.name] = arr
                self.buffers[f.name] = DataBuffer(f.name, self.dtype, (n,),
                                                  data=arr)
            self.host_sections.append(
                (self.op.artifact.sections[len(self.host_sections)],
                 time.perf_counter() - t0, n * len(c.eqs)))

    def _prange(self, pdim) -> Tuple[int, int]:
        lo = int(self.env.get(pdim.name + "_m", 0))
        hi = int(self.env.get(pdim.name + "_M", -1))
        return lo, hi

    # -- device state -------------------------------------------------------------------

    def _upload(self):
        torch = self._torch
        tdt = torch.float32 if self.dtype == "f32" else torch.float64
        self.dev: Dict[str, "torch.Tensor"] = {}
        dev = "cpu" if self.dry else "cuda:%d" % self.device
        self.no_upload = self._overwritten_sparse()
        for f in self.op.functions.values():
            if f.kind == "coordinates":
                continue
            host = self._window(f, self.buffers[f.name].data)
            t = torch.empty(host.shape, dtype=tdt, device=dev)
            self.dev[f.name] = t
        self.h2d_bytes = self._copy_inputs()

    def _copy_inputs(self) -> int:
        """Host -> device copies of every input buffer (pinned host memory,
        current stream, asynchronous: they proceed while the host builds the
        plan; the library's prepare/launch run on the same stream). Sparse
        outputs whose every row the run overwrites are not uploaded."""
        torch = self._torch
        nbytes = 0
        dead = getattr(self, "dead", {})
        for name, t in self.dev.items():
            if name in self.no_upload:
                continue
            f = self.op.functions[name]
            host = self._window(f, self.buffers[name].data)
            if name in dead and host.flags.c_contiguous:
                nbytes += self._copy_live(t, host, *dead[name])
                continue
            t.copy_(torch.from_numpy(np.ascontiguousarray(host)),
                    non_blocking=not self.dry)
            nbytes += t.numel() * t.element_size()
        return nbytes

    def _copy_live(self, t, host, slot: int, lo, hi) -> int:
        """Upload of a time function whose time slot ``slot`` is dead on
        entry inside the box lo..hi (storage coordinates): the other slots
        whole, that slot's halo shell only (sc_upload_shell reads the
        page-locked host array in place); returns the bytes moved."""
        torch = self._torch
        nbytes = 0
        esz = t.element_size()
        for s in range(t.shape[0]):
            if s != slot:
                t[s].copy_(torch.from_numpy(host[s]), non_blocking=True)
                nbytes += t[s].numel() * esz
        ext = (C.c_int64 * 3)(*t.shape[1:])
        clo = (C.c_int32 * 3)(*lo)
        chi = (C.c_int32 * 3)(*hi)
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream().cuda_stream
            rc = rt.load_library().sc_upload_shell(
                C.c_void_p(t[slot].data_ptr()),
                C.c_void_p(host[slot].ctypes.data), ext, clo, chi, esz,
                C.c_void_p(stream))
        if rc < 0:
            raise BackendError(rt.last_error())
        if rc != 0:      # pageable host memory: the whole slot
            t[slot].copy_(torch.from_numpy(host[slot]), non_blocking=True)
            return nbytes + t[slot].numel() * esz
        box = int(np.prod([h - l + 1 for l, h in zip(lo, hi)]))
        return nbytes + (t[slot].numel() - box) * esz

    def _dead_on_entry(self) -> dict:
        """Time slots whose loop box the first time step overwrites before
        any stage reads them (u[t_m + 1] of a leapfrog update: the stencil
        writes the whole box, injections add to it afterwards). A prepared
        run that is reused uploads only the halo shell of such a slot:
        {function: (slot, lo, hi)} in storage coordinates. Decided from the
        plan's stage order at step t_m; anything unusual (windows, guards,
        sub-sampled or shifted targets, functions without a halo frame)
        keeps the full upload. ``SC_FULL_UPLOAD=1`` disables it."""
        if self.dry or self.xwin is not None or self.t_M < self.t_m or \
                self.grid.ndim != 3 or os.environ.get("SC_FULL_UPLOAD"):
            return {}
        plan = self.plan
        names = {v: k for k, v in self.field_ids.items()}
        # (field, slot) -> first access at step t_m: None = read, else the
        # storage offset of the loop box a full write covers
        first: Dict[Tuple[int, int], Optional[tuple]] = {}

        def touch(field, tshift, off=None):
            fd = plan.fields[field]
            if not fd.has_time or fd.nslots < 2:
                return
            first.setdefault((field, (self.t_m + tshift) % fd.nslots), off)

        for i in range(plan.nstages):
            code = plan.stages[i]
            if code >= 100:
                sp = plan.sparse[code - 100]
                touch(sp.field, sp.field_tshift)
                continue
            d = plan.dense[code]
            if d.fast_kind == 3:            # fused TTI: p, r at t, t-1 -> t+1
                H = d.so // 2
                for k in (0, 1):
                    touch(d.tti_fields[k], 0)
                    touch(d.tti_fields[k], -1)
                for k in (0, 1):
                    touch(d.tti_fields[k], 1,
                          (H, H, H) if d.tguard == 0 else None)
                continue
            plain = d.tguard == 0
            for j in range(d.nloads):
                ld = d.loads[j]
                plain = plain and ld.tdiv == 1
                touch(ld.field, ld.tshift)
            tg = d.target
            whole = plain and tg.tdiv == 1
            touch(tg.field, tg.tshift,
                  tuple(tg.off[k] for k in range(3)) if whole else None)
        out = {}
        for (field, slot), off in first.items():
            name = names.get(field)
            f = self.op.functions.get(name) if name else None
            if off is None or f is None or name in out or \
                    f.kind != "timefunction":
                continue
            lo = [l + o for l, o in zip(self.lo, off)]
            hi = [h + o for h, o in zip(self.hi, off)]
            ext = tuple(self.dev[name].shape[1:])
            if any(l < 0 or h >= e or h < l for l, h, e in zip(lo, hi, ext)):
                continue
            out[name] = (slot, lo, hi)
        return out

    def _overwritten_sparse(self) -> set:
        """Sparse functions written (not incremented) by an interpolation at
        every row: rows t + k for t in [t_m, t_M] cover the whole time axis."""
        out = set()
        for c in self.timed:
            if c.guards or any(d.kind == "space" for d in c.dims) or \
                    c.fused is not None:
                continue
            for e in c.eqs:
                f = e.lhs.func
                if f.kind != "sparsetimefunction" or e.is_increment:
                    continue
                k = _time_shift(e.lhs)
                nt = self.buffers[f.name].data.shape[0]
                if self.t_m + k <= 0 and self.t_M + k >= nt - 1:
                    out.add(f.name)
        # never skip a function that is also read
        for c in self.timed + self.post:
            for e in c.eqs:
                for acc in _deep_accesses(e.rhs):
                    out.discard(acc.func.name)
        return out

    # -- reuse across applies (Operator.apply) -----------------------------------

    def signature(self) -> tuple:
        return tuple(sorted((k, tuple(b.data.shape), str(b.data.dtype))
                            for k, b in self.buffers.items()
                            if k in self.op.functions))

    def inputs_unchanged(self, buffers: Dict[str, DataBuffer]) -> bool:
        """True when every host value that fed a per-point table (coordinates,
        fields read by injected expressions) is bitwise what this run saw."""
        for name, idx, vals in self.reads:
            if name in self.tables or name not in buffers:
                if name in self.tables:
                    continue
                return False
            got = buffers[name].data[idx]
            if got.shape != vals.shape or \
                    got.tobytes() != vals.tobytes():
                return False
        return True

    def rebind(self, buffers: Dict[str, DataBuffer]) -> int:
        """Point a prepared run at the caller's (same-shaped) buffers and
        re-upload their contents; the hoisted tables reappear in
        ``buffers`` as the reference exposes them."""
        self.buffers = buffers
        for name, arr in self.tables.items():
            buffers[name] = DataBuffer(name, self.dtype, arr.shape, data=arr)
        self.h2d_bytes = self._copy_inputs()
        return self.h2d_bytes

    def revalidate(self) -> bool:
        """Re-check the fused kernels' data-dependent preconditions (the
        acoustic kernel's reciprocal operand range) on the re-uploaded
        buffers, on the upload stream; False: prepare afresh."""
        prep = getattr(self, "_prepared", None)
        if prep is None:
            return True
        with self._torch.cuda.device(self.device):
            stream = self._torch.cuda.current_stream().cuda_stream
            return prep.revalidate(stream)

    def _xaxis(self, f) -> Optional[int]:
        if self.xwin is None or f.kind not in ("function", "timefunction"):
            return None
        return 1 if f.kind == "timefunction" else 0

    def _window(self, f, host):
        ax = self._xaxis(f)
        if ax is None or host.shape[ax] == self.xwin[1] - self.xwin[0]:
            return host                  # not windowed / already a window
        sl = [slice(None)] * host.ndim
        sl[ax] = slice(*self.xwin)
        return host[tuple(sl)]

    def _field_index(self, name: str) -> int:
        if name not in self.field_ids:
            if len(self.field_ids) >= rt.MAX_FIELDS:
                raise BackendError("too many fields")
            self.field_ids[name] = len(self.field_ids)
        return self.field_ids[name]

    def _fill_fields(self, plan):
        for name, i in self.field_ids.items():
            f = self.op.functions[name]
            t = self.dev[name]
            fd = plan.fields[i]
            fd.data = t.data_ptr()
            for k, e in enumerate(t.shape):
                fd.ext[k] = e
            fd.ndim = t.dim()
            fd.has_time = 1 if f.kind == "timefunction" else 0
            fd.nslots = f.time_dim.modulo if f.is_modulo_time else 0
        plan.nfields = len(self.field_ids)

    def _build_plan(self, clusters=None):
        """The C plan of one device phase: the main t loop (``clusters``
        None: self.timed; sets self.plan and the per-stage lists), or a
        time-inner nest run after it (returns the plan record)."""
        main = clusters is None
        if main:
            clusters = self.timed
        plan = rt.ScPlan()
        g = self.grid
        plan.dtype = 0 if self.dtype == "f32" else 1
        plan.ndim = g.ndim
        self.lo = [int(self.env[d.name + "_m"]) for d in g.dimensions]
        self.hi = [int(self.env[d.name + "_M"]) for d in g.dimensions]
        self.xshift = 0
        if self.xwin is not None:
            self.xshift = self.xwin[0]
            self.lo[0] -= self.xshift
            self.hi[0] -= self.xshift
        for d in range(g.ndim):
            plan.lo[d], plan.hi[d] = self.lo[d], self.hi[d]
        plan.t_m, plan.t_M = self.t_m, self.t_M
        if main:
            self.field_ids: Dict[str, int] = {}
            self.written: List[str] = []
            self.fast_used: List[int] = []
        stages: List[int] = []
        stage_names: List[str] = []
        stage_points: List[int] = []
        nd = ns = 0
        # per-step point counts as the reference's interpreter reports them
        # (every statement, scalar temporaries included, counts its
        # iteration points; interpreter.py:231, 302): (guard, count)
        ref_points: List[Tuple[int, int]] = []
        box = max(int(np.prod([h - l + 1 for l, h in zip(self.lo, self.hi)])), 0)
        for c in clusters:
            if any(d.kind == "space" for d in c.dims) or c.fused is not None:
                ref_points.append((_guard(c), len(c.eqs) * box))
            else:
                pdim = [d for d in c.dims if d.kind == "sparse"]
                lo_, hi_ = self._prange(pdim[0]) if pdim else (0, 0)
                ref_points.append((_guard(c),
                                   len(c.eqs) * max(hi_ - lo_ + 1, 0)))
        for c in clusters:
            if c.fused is not None:
                if nd >= rt.MAX_DENSE:
                    raise BackendError("too many dense statements")
                self._tti_stage(plan.dense[nd], c.fused[1])
                stages.append(nd)
                stage_names.append("dense:tti")
                stage_points.append(max(int(np.prod(
                    [h - l + 1 for l, h in zip(self.lo, self.hi)])), 0))
                nd += 1
            elif any(d.kind == "space" for d in c.dims):
                progs = compile_dense(c.eqs, self.env, self.dtype)
                for prog in progs:
                    if nd >= rt.MAX_DENSE:
                        raise BackendError("too many dense statements")
                    self._dense_stage(plan.dense[nd], prog, _guard(c))
                    stages.append(nd)
                    stage_names.append("dense:" + prog.target.func)
                    npts = int(np.prod([h - l + 1 for l, h in
                                        zip(self.lo, self.hi)]))
                    stage_points.append(max(npts, 0))
                    nd += 1
            else:
                if c.guards:
                    raise BackendError("sub-sampled sparse statements are not "
                                       "supported by the B200 backend")
                for group in _sparse_groups(c):
                    if ns >= rt.MAX_SPARSE:
                        raise BackendError("too many sparse statements")
                    n = self._sparse_stage(plan.sparse[ns], c, group)
                    stages.append(100 + ns)
                    stage_names.append("sparse:%d" % ns)
                    stage_points.append(n)
                    ns += 1
        plan.ndense, plan.nsparse = nd, ns
        if len(stages) > rt.MAX_STAGES:
            raise BackendError("too many stages per time step")
        plan.nstages = len(stages)
        for i, s in enumerate(stages):
            plan.stages[i] = s
        self._fill_fields(plan)
        if not main:
            return {"plan": plan, "stage_names": stage_names,
                    "stage_points": stage_points, "ref_points": ref_points,
                    "prepared": None, "main": False}
        self.plan, self.ref_points = plan, ref_points
        self.post_plans = [self._build_plan([c]) for c in self.post]
        self.stage_names, self.stage_points = stage_names, stage_points
        self._fill_fields(plan)

    # dense stage --------------------------------------------------------------------

    def _check_load_bounds(self, func: str, ld, guard: int = 0):
        f = self.op.functions[func]
        ext = self.dev[func].shape
        sp = 1 if f.kind == "timefunction" else 0
        for d, (a, b) in enumerate(_ld_range(ld, self.lo, self.hi)):
            if b < a:
                continue
            if a < 0 or b >= ext[sp + d]:
                raise BoundsError("%s slice [%d, %d) out of range [0, %d) "
                                  "along axis %d" % (func, a, b + 1,
                                                     ext[sp + d], sp + d))
        if f.kind == "timefunction" and not f.is_modulo_time:
            ts = [t for t in range(self.t_m, self.t_M + 1)
                  if guard <= 1 or t % guard == 0] if guard > 1 else \
                [self.t_m, self.t_M]
            for t in ts[:1] + ts[-1:]:
                v = (t // ld.tdiv if ld.tdiv > 1 else t) + (ld.tshift or 0)
                if not 0 <= v < ext[0]:
                    raise BoundsError("%s index %d out of range [0, %d) along "
                                      "axis 0" % (func, v, ext[0]))

    def _dense_stage(self, d: rt.ScDense, prog: DenseProgram, guard: int = 0):
        d.tguard = guard
        # loop blocking along x (reference block={"x": ...}, iet.py:377-423):
        # x planes per CTA chunk of the fused kernels
        blk = self.op.block or {}
        dims = [dd.name for dd in self.grid.dimensions]
        d.xblock = int(blk.get(dims[0], 0)) if self.grid.ndim == 3 else 0
        # y/z blocking (reference iet.py:377-423) shapes the generated
        # kernels' thread blocks: innermost axis and the next one
        d.iblock = int(blk.get(dims[-1], 0))
        d.jblock = int(blk.get(dims[-2], 0)) if self.grid.ndim >= 2 else 0
        if self.t_M >= self.t_m:
            for ld in prog.loads + [prog.target]:
                self._check_load_bounds(ld.func, ld, guard)
        ops = (rt.ScOp * max(1, len(prog.ops)))()
        for i, (o, a1, a2, a3) in enumerate(prog.ops):
            ops[i].op, ops[i].dst, ops[i].a, ops[i].b = o, a1, a2, a3
        loads = (rt.ScLoad * max(1, len(prog.loads)))()
        for i, ld in enumerate(prog.loads):
            loads[i].field = self._field_index(ld.func)
            loads[i].tshift = ld.tshift or 0
            loads[i].tdiv = ld.tdiv
            for k, v in enumerate(ld.offs):
                loads[i].off[k] = v
        consts = (C.c_double * max(1, len(prog.consts)))(*prog.consts)
        self._keep += [ops, loads, consts]
        d.nops, d.nloads, d.nconsts = len(prog.ops), len(prog.loads), \
            len(prog.consts)
        d.out_reg, d.nregs = prog.out, prog.nregs
        d.ops = C.cast(ops, C.POINTER(rt.ScOp))
        d.loads = C.cast(loads, C.POINTER(rt.ScLoad))
        d.consts = C.cast(consts, C.POINTER(C.c_double))
        d.target.field = self._field_index(prog.target.func)
        d.target.tshift = prog.target.tshift or 0
        d.target.tdiv = prog.target.tdiv
        for k, v in enumerate(prog.target.offs):
            d.target.off[k] = v
        self.written.append(prog.target.func)
        d.fast_kind = 0
        fast = self._try_fast(prog)
        if fast is not None:
            kind, so, names, damp, k = fast
            d.fast_kind, d.so, d.has_damp = kind, so, int(damp)
            d.u_field = self._field_index(names["u"])
            d.m_field = self._field_index(names["m"])
            d.damp_field = self._field_index(names["damp"]) if damp else \
                d.m_field
            kc = (C.c_double * len(k))(*k)
            self._keep.append(kc)
            d.fast_consts = C.cast(kc, C.POINTER(C.c_double))
            d.nfast_consts = len(k)
            self.fast_used.append(kind)

    def _tti_stage(self, d: rt.ScDense, roles: dict):
        """Fused TTI step (csrc/tti.cu): p/r updates with rotated second
        derivatives; temporaries g_p, g_r in device scratch."""
        from ..symbolic.fd import centered_weights
        p = roles["p"]
        so = p.space_order
        d.xblock = int((self.op.block or {}).get(
            self.grid.dimensions[0].name, 0))
        H = so // 2
        names = [roles[k].name for k in ("p", "r", "m", "damp", "epsilon",
                                         "delta", "theta", "phi")]
        ext = tuple(self.dev[p.name].shape[1:])
        for n in names:
            f = self.op.functions[n]
            sh = tuple(self.dev[n].shape[1:] if f.kind == "timefunction"
                       else self.dev[n].shape)
            if sh != ext or f.halo != H or f.padding:
                raise BackendError("TTI fields must share extents and the "
                                   "so/2 halo (%s)" % n)
            if f.kind == "timefunction" and f.time_dim.modulo != 3:
                raise BackendError("TTI needs time_order 2 (3 slots)")
        for dd in range(3):
            if self.lo[dd] < 0 or self.hi[dd] > ext[dd] - 2 * H - 1:
                raise BoundsError("%s_M=%d outside the TTI reach" %
                                  ("xyz"[dd], self.hi[dd]))
        if "dt" not in self.env:
            raise BackendError("unbound symbol 'dt'")
        dt = float(self.env["dt"])
        h = [float(self.env["h_" + c]) for c in "xyz"]
        w1 = centered_weights(so // 2, 1)
        w2 = centered_weights(so, 2)
        k = [1 / x for x in h] + [1 / (x * x) for x in h] + \
            [1 / (dt * dt), 1 / (2 * dt)]
        k += [float(w1.get(i, 0)) for i in range(1, 6)]
        k += [float(w2.get(i, 0)) for i in range(0, 9)]
        kc = (C.c_double * len(k))(*k)
        torch = self._torch
        # g_p, g_r; in f32 also the four hoisted per-point coefficients
        # the TMA kernels read instead of m, damp, epsilon, delta
        nscr = 6 if self.dtype == "f32" else 2
        g = [torch.zeros(ext, dtype=self.dev[p.name].dtype,
                         device=self.dev[p.name].device) for _ in range(nscr)]
        self._keep += [kc] + g
        d.fast_kind, d.so = 3, so
        d.fast_consts = C.cast(kc, C.POINTER(C.c_double))
        d.nfast_consts = len(k)
        for i, n in enumerate(names):
            d.tti_fields[i] = self._field_index(n)
        for i, gt in enumerate(g):
            d.scratch[i] = gt.data_ptr()
        d.nops = 0
        self.written += [names[0], names[1]]
        self.fast_used.append(3)

    def _try_fast(self, prog: DenseProgram):
        if any(ld.tdiv != 1 for ld in prog.loads + [prog.target]):
            return None
        """Route to the fused acoustic kernel when its op sequence equals
        the program (backend/fastpath.py)."""
        g = self.grid
        if g.ndim != 3 or prog.target.tshift != 1:
            return None
        u = self.op.functions[prog.target.func]
        if not u.is_modulo_time or u.time_dim.modulo != 3:
            return None
        so = 2 * u.halo
        if so < 2 or so > 16 or u.padding:
            return None
        if any(self.hi[d] < self.lo[d] for d in range(3)):
            return None
        dense_in = sorted({ld.func for ld in prog.loads
                           if ld.func != u.name})
        if len(dense_in) not in (1, 2):
            return None
        ext = self.dev[u.name].shape[1:]
        for nm in dense_in:
            if tuple(self.dev[nm].shape) != tuple(ext):
                return None
        if (ext[2] * self.np_t().itemsize) % 16:
            return None
        trace = program_trace(prog)
        cands = [(dense_in[0], None)] if len(dense_in) == 1 else \
            [(dense_in[0], dense_in[1]), (dense_in[1], dense_in[0])]
        for m, damp in cands:
            names = {"u": u.name, "m": m, "damp": damp}
            hit = match_acoustic(prog, trace, so, self.env, names, self.dtype,
                                 damp is not None)
            if hit is not None:
                return hit[0], so, names, damp is not None, hit[1]
        return None

    # sparse stage -------------------------------------------------------------------

    def _sparse_stage(self, s: rt.ScSparse, c, mains) -> int:
        pdim = [d for d in c.dims if d.kind == "sparse"][0]
        lo, hi = self._prange(pdim)
        sp_decl = [f for f in self.op.functions.values()
                   if f.kind == "sparsetimefunction" and
                   f.point_dim.name == pdim.name]
        if not sp_decl:
            raise BackendError("no sparse function iterates %s" % pdim.name)
        sp_decl = sp_decl[0]
        if lo != 0 or hi != sp_decl.npoint - 1:
            raise BackendError("partial sparse ranges (%s_m/%s_M) are not "
                               "supported" % (pdim.name, pdim.name))
        n = hi - lo + 1
        arrays = self._arrays()
        arrays.update(self.tables)
        xoff = {}
        if self.xwin is not None:
            for f in self.op.functions.values():
                ax = self._xaxis(f)
                if ax is not None and arrays[f.name].shape[ax] == \
                        self.xwin[1] - self.xwin[0]:
                    xoff[f.name] = self.xwin[0]
        ev = SparseEvaluator(self.env, self.dtype, n, arrays, {}, pdim.name, 0,
                             xoff, reads=self.reads)
        temps = [e for e in c.eqs if e.lhs.func.kind == "temp"]
        varying = {}
        for e in temps:
            if e.lhs.indices:
                raise BackendError("array temporaries in sparse loops")
            if _time_varying(e.rhs):
                varying[e.lhs.func.name] = e.rhs
                continue
            ev.temps[e.lhs.func.name] = ev.ev(e.rhs)
        # a statement whose whole right-hand side is a time-varying CSE temp
        # (the same injected value added to several fields) evaluates that
        # temp's expression with the same fold: inline it
        inl = []
        for e in mains:
            if isinstance(e.rhs, Access) and e.rhs.func.kind == "temp" and \
                    not e.rhs.indices and e.rhs.func.name in varying:
                e = LoweredEq(e.lhs, varying[e.rhs.func.name], e.is_increment,
                              e.region, e.dims, e.dspace)
            inl.append(e)
        mains = inl
        incs = all(e.is_increment for e in mains)
        if incs:
            field = mains[0].lhs.func
            if field.kind != "timefunction" or \
                    any(e.lhs.func is not field for e in mains):
                raise BackendError("unsupported injection target")
            corners = [(e.lhs, e.rhs) for e in mains]
            s.kind = 0
        else:
            if len(mains) != 1:
                raise BackendError("unsupported sparse cluster")
            eq = mains[0]
            if eq.lhs.func.kind != "sparsetimefunction" or eq.is_increment:
                raise BackendError("unsupported interpolation target")
            terms = list(eq.rhs.children) if isinstance(eq.rhs, Add) \
                else [eq.rhs]
            corners = []
            field = None
            for tm in terms:
                fa = [a for a in _factor_list(tm) if isinstance(a, Access) and
                      a.func.kind == "timefunction"]
                if len(fa) != 1:
                    raise BackendError("interpolation term must read one "
                                       "field: %r" % (tm,))
                if field is None:
                    field = fa[0].func
                elif fa[0].func is not field:
                    raise BackendError("interpolation mixes fields")
                corners.append((fa[0], tm))
            s.kind = 1
        if len(corners) > rt.MAX_CORNERS or \
                (s.kind == 1 and len(corners) not in (1, 2, 4, 8)):
            raise BackendError("unsupported corner count %d" % len(corners))
        s.npoint, s.ncorner, s.ndim = n, len(corners), self.grid.ndim
        s.field = self._field_index(field.name)
        # corner indices: evaluated exactly as resolve_indices does
        tshift = None
        idx_all = []
        for acc, _ in corners:
            tk = _time_shift(acc)
            if tshift is None:
                tshift = tk
            elif tk != tshift:
                raise BackendError("corners at different time levels")
            ii = [ev.index(i) for i in acc.indices[1:]]
            ii[0] = ii[0] - self.xshift
            idx_all.append(ii)
        s.field_tshift = tshift
        nd = self.grid.ndim
        base = [np.asarray(idx_all[0][dd], np.int64) for dd in range(nd)]
        ext = self.dev[field.name].shape
        # every corner is base + a constant offset; bounds then follow from
        # the base's extremes (one pass per corner and dimension)
        bmin = [int(b.min()) if n else 0 for b in base]
        bmax = [int(b.max()) if n else 0 for b in base]
        for ci, idx in enumerate(idx_all):
            for dd in range(nd):
                col = idx[dd]
                d0 = int(col[0] - base[dd][0]) if n else 0
                if n and not np.array_equal(col - base[dd], np.broadcast_to(
                        np.int64(d0), (n,))):
                    raise BackendError("corner offsets vary across points")
                s.delta[ci][dd] = d0
                if n and (bmin[dd] + d0 < 0 or bmax[dd] + d0 >= ext[1 + dd]):
                    bad = (col < 0) | (col >= ext[1 + dd])
                    raise BoundsError("%s index %d out of range [0, %d) along "
                                      "axis %d" % (field.name, col[bad][0],
                                                   ext[1 + dd], 1 + dd))
        base32 = self._to_dev(np.stack(base).astype(np.int32))
        self._keep.append(base32)
        s.base = base32.data_ptr()
        if s.kind == 0:
            lin = np.zeros((len(corners), n), np.int64)
            for ci, idx in enumerate(idx_all):
                for dd in range(self.grid.ndim):
                    lin[ci] = lin[ci] * ext[1 + dd] + idx[dd]
            flat = lin.T.reshape(-1)
            s.serial = int(len(np.unique(flat)) != flat.size)
        # factor programs: fold order of evaluate() (expr.py:461-465)
        tables: List[np.ndarray] = []
        table_ids: Dict[str, int] = {}
        sparse_name = None
        for ci, (acc, expr) in enumerate(corners):
            lead = 1.0                  # leading Python-float product
            items = []
            seen_np = False
            for fx in _factor_list(expr):
                kind, arg, val = self._classify(fx, acc, field, ev, n)
                if kind == "py":
                    if not seen_np:
                        lead = lead * val
                    elif np.ndim(val):
                        items.append((FAC_TABLE, self._table(
                            val, tables, table_ids, "py:" + repr(fx), n), 0.0))
                    else:
                        items.append((FAC_CONST, 0, float(self.np_t(val))))
                    continue
                if not seen_np and np.ndim(lead):
                    items.append((FAC_TABLE, self._table(
                        lead, tables, table_ids, "lead:%d" % ci, n), 0.0))
                    lead = 1.0
                seen_np = True
                if kind == FAC_SPARSE:
                    if sparse_name is None:
                        sparse_name, s.sparse_tshift = arg
                    elif (sparse_name, s.sparse_tshift) != arg:
                        raise BackendError("several sparse operands")
                    arg = 0
                elif kind == FAC_TABLE:
                    arg = self._table(val, tables, table_ids, repr(fx), n)
                items.append((kind, arg, 0.0))
            if not seen_np:
                raise BackendError("sparse term without array operand")
            if len(items) > rt.MAX_FACTORS:
                raise BackendError("too many factors")
            for k, (kind, arg, cv) in enumerate(items):
                s.fac_kind[ci][k], s.fac_arg[ci][k] = kind, arg
                s.fac_const[ci][k] = cv
            s.nfac[ci] = len(items)
            s.lead[ci] = float(self.np_t(lead))
        if len(tables) > rt.MAX_TABLES:
            raise BackendError("too many per-point tables")
        for i, tb in enumerate(tables):
            t = self._to_dev(tb)
            self._keep.append(t)
            s.tables[i] = t.data_ptr()
        if s.kind == 1:
            sparse_name = mains[0].lhs.func.name
            s.sparse_tshift = _time_shift(mains[0].lhs)
            self.written.append(sparse_name)
        if sparse_name is None:
            raise BackendError("sparse cluster reads no sparse function")
        st = self.dev[sparse_name]
        s.sparse = st.data_ptr()
        s.sparse_nt = st.shape[0]
        for t in (self.t_m, self.t_M):
            v = t + s.sparse_tshift
            if self.t_M >= self.t_m and not 0 <= v < st.shape[0]:
                raise BoundsError("%s index %d out of range [0, %d) along "
                                  "axis 0" % (sparse_name, v, st.shape[0]))
        if s.kind == 0:
            self.written.append(field.name)
        return n * len(corners)

    def _to_dev(self, arr: np.ndarray):
        t = self._torch.from_numpy(np.ascontiguousarray(arr).copy())
        if self.dry:
            return t
        # pinned staging + asynchronous copy: a pageable copy would wait for
        # the (asynchronous) buffer uploads queued on the same stream
        h = t.pin_memory()
        self._keep.append(h)
        return h.to("cuda:%d" % self.device, non_blocking=True)

    def _table(self, values, tables, ids, key, n) -> int:
        if key not in ids:
            ids[key] = len(tables)
            tables.append(np.ascontiguousarray(np.broadcast_to(
                np.asarray(values).astype(self.np_t), (n,))))
        return ids[key]

    def _classify(self, fx: Expr, corner_acc: Access, field, ev, n):
        """Factor kind: sparse operand, dense field at the corner, Python
        float (uniform or per point), or a per-point time-invariant dtype
        value evaluated on the host with the oracle's semantics."""
        if isinstance(fx, Access) and fx.func.kind == "sparsetimefunction":
            return FAC_SPARSE, (fx.func.name, _time_shift(fx)), None
        if isinstance(fx, Access) and fx.func is field:
            if fx.indices[1:] != corner_acc.indices[1:] or \
                    _time_shift(fx) != _time_shift(corner_acc):
                raise BackendError("field read at a different corner")
            return FAC_FIELD, 0, None
        if _time_varying(fx):
            raise BackendError("unsupported time-varying factor %r" % (fx,))
        v = ev.ev(fx)
        if v.kind == "py":
            return "py", 0, v.v
        return FAC_TABLE, 0, v.v

    # -- execution ------------------------------------------------------------------

    # -- execution ------------------------------------------------------------------

    def run(self, profile: bool = True, early_download: bool = False) -> dict:
        """Execute t_m..t_M. ``profile`` times every stage launch with CUDA
        events (per-section report); otherwise only the whole loop. Time-
        inner nests (``post_plans``) run after the main loop, each as its
        own section, as the reference schedules them."""
        if self.dry:
            raise BackendError("a dry plan cannot run")
        torch = self._torch
        main = {"plan": self.plan, "stage_names": self.stage_names,
                "stage_points": self.stage_points,
                "ref_points": self.ref_points, "main": True,
                "prepared": getattr(self, "_prepared", None)}
        recs = [main] + self.post_plans
        walls = []
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream()
            for r in recs:
                plan = r["plan"]
                plan.stream = stream.cuda_stream
                t0 = time.perf_counter()
                if self.t_M >= self.t_m and plan.nstages:
                    if r["prepared"] is None:
                        plan.profile = 0        # capture the graph
                        r["prepared"] = rt.PreparedRun(plan)
                    plan.profile = 1 if profile else 0
                    if r is main:
                        self._arm_early_download(r["prepared"], early_download)
                    r["prepared"].launch(plan)
                walls.append(time.perf_counter() - t0)
        self._prepared = main["prepared"]
        report = {}
        for name, sec, pts in self.host_sections:
            report[name] = {"time": sec, "points": pts}
        if self.t_M >= self.t_m:
            nsteps = self.t_M - self.t_m + 1
            for k, r in enumerate(recs):
                if r["plan"].nstages:
                    plan = r["plan"]
                    idx = len(report)
                    secs = self.op.artifact.sections
                    name = secs[idx] if idx < len(secs) else "section%d" % idx
                    pts = sum(n for t in range(self.t_m, self.t_M + 1)
                              for g, n in r["ref_points"]
                              if g <= 1 or t % g == 0)
                    report[name] = {
                        "time": plan.total_ms / 1e3, "points": pts,
                        "stage_points": nsteps * sum(r["stage_points"]),
                        "wall": walls[k],
                        "stages": {n: plan.stage_ms[i] / 1e3
                                   for i, n in enumerate(r["stage_names"])},
                        "launches": int(plan.launches),
                        "fast_path": any(plan.dense[i].fast_kind
                                         for i in range(plan.ndense)),
                        "dense_exec": [("interpreter", "generated", "acoustic",
                                        "tti")[plan.dense[i].exec_kind]
                                       for i in range(plan.ndense)]}
        self.report = report
        return report

    def _arm_early_download(self, prepared, want: bool) -> None:
        """Rows of an interpolated sparse function are final as soon as
        their time step is done: let the launch copy all but the last few
        of them to the caller's (page-locked) array while the loop still
        runs (sc_early_download); download() then copies the rest.
        ``SC_NO_EARLY_D2H=1`` switches it off."""
        self._early = None
        nsteps = self.t_M - self.t_m + 1
        if not want or self.xwin is not None or self.post_plans or \
                nsteps < 64 or os.environ.get("SC_NO_EARLY_D2H"):
            prepared.early_download(0, 0, 0, 0)
            return
        best = None
        for c in self.timed:
            if c.guards or any(d.kind == "space" for d in c.dims) or \
                    c.fused is not None:
                continue
            for e in c.eqs:
                f = e.lhs.func
                if f.kind != "sparsetimefunction" or e.is_increment or \
                        f.name not in self.dev:
                    continue
                t = self.dev[f.name]
                if best is None or t.numel() > best[1].numel():
                    best = (f.name, t, _time_shift(e.lhs))
        # one writer per function, and nothing else in the loop touches it
        if best is not None:
            writers = sum(1 for c in self.timed for e in c.eqs
                          if e.lhs.func.name == best[0])
            readers = any(acc.func.name == best[0] for c in self.timed
                          for e in c.eqs for acc in _deep_accesses(e.rhs))
            if writers != 1 or readers:
                best = None
        host = self.buffers[best[0]].data if best is not None else None
        if best is None or not host.flags.c_contiguous or \
                not self._torch.from_numpy(host).is_pinned():
            prepared.early_download(0, 0, 0, 0)
            return
        name, t, shift = best
        t_split = self.t_M - max(8, nsteps // 16) + 1
        rows = min(max(t_split + shift, 0), t.shape[0])
        nbytes = rows * (t.numel() // t.shape[0]) * t.element_size()
        if rows <= 0 or not prepared.early_download(
                t_split, t.data_ptr(), host.ctypes.data, nbytes):
            prepared.early_download(0, 0, 0, 0)
            return
        self._early = (name, rows)

    def step(self, t: int) -> None:
        """Launch time step ``t`` asynchronously on the current stream
        (host-driven loops: slab runs exchange ghost planes between steps)."""
        if self.dry:
            raise BackendError("a dry plan cannot run")
        torch = self._torch
        if self.post_plans:
            raise BackendError("step-driven runs do not support time-inner "
                               "loop nests")
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream()
            if getattr(self, "_prepared", None) is None:
                self.plan.stream = stream.cuda_stream
                self.plan.profile = 1        # no graph capture for step mode
                self._prepared = rt.PreparedRun(self.plan)
            self._prepared.step(t, stream.cuda_stream)

    def prepared(self):
        """The C-side prepared run for host-driven and library-driven
        (sc_multi_run) loops: stage by stage, no whole-loop graph."""
        prep = getattr(self, "_prepared", None)
        if prep is None:
            if self.dry:
                raise BackendError("a dry plan cannot run")
            torch = self._torch
            with torch.cuda.device(self.device):
                self.plan.stream = torch.cuda.current_stream().cuda_stream
                self.plan.profile = 1
                prep = self._prepared = rt.PreparedRun(self.plan)
        return prep

    # parts of a time step (what: 1 dense, 2 injection, 4 interpolation)
    DENSE, INJECT, INTERP = 1, 2, 4

    def can_split(self) -> bool:
        """Whether every stage can run in parts (fused acoustic kernel,
        hoisted-prefix sparse kernels)."""
        try:
            self.step_part(self.t_m, 0)
            return True
        except BackendError:
            return False

    def step_part(self, t: int, what: int, x_lo: int = 0, x_hi: int = -1,
                  p_lo: int = 0, p_hi: int = 1 << 30) -> None:
        """Launch part of time step ``t`` on the current stream: the dense
        stages over loop x planes [x_lo, x_hi] (global loop coordinates)
        and/or the sparse stages over points [p_lo, p_hi). Multi-GPU slabs
        use it to finish boundary planes before their ghost exchange and
        compute the interior while the planes travel (backend/slab.py)."""
        prep = getattr(self, "_prepared", None)
        if prep is None:
            if self.dry:
                raise BackendError("a dry plan cannot run")
            torch = self._torch
            with torch.cuda.device(self.device):
                self.plan.stream = torch.cuda.current_stream().cuda_stream
                self.plan.profile = 1        # no graph capture for step mode
                prep = self._prepared = rt.PreparedRun(self.plan)
        # hot path of host-driven loops: no device context switch
        stream = self._torch.cuda.current_stream(self.device).cuda_stream
        prep.step_part(t, stream, x_lo - self.xshift, x_hi - self.xshift,
                       p_lo, p_hi, what)

    def close(self):
        """Release the prepared C-side run (device programs, CUDA graph)."""
        p = getattr(self, "_prepared", None)
        if p is not None:
            p.close()
            self._prepared = None
        for r in getattr(self, "post_plans", ()):
            if r["prepared"] is not None:
                r["prepared"].close()
                r["prepared"] = None

    def download(self, xrange: Optional[Tuple[int, int]] = None):
        """Copy written functions back into the caller's buffers. With a
        window, ``xrange`` (global storage planes) limits dense write-back to
        the planes this run owns."""
        torch = self._torch
        self.d2h_bytes = 0
        for name in dict.fromkeys(self.written):
            t = self.dev[name]
            f = self.op.functions[name]
            host = self._window(f, self.buffers[name].data)
            ax = self._xaxis(f)
            if ax is not None and xrange is not None:
                sl = [slice(None)] * t.dim()
                sl[ax] = slice(xrange[0] - self.xwin[0], xrange[1] - self.xwin[0])
                t, host = t[tuple(sl)], host[tuple(sl)]
            early = getattr(self, "_early", None)
            if early is not None and early[0] == name:
                # rows [0, early[1]) arrived while the loop ran
                self.d2h_bytes += early[1] * (t.numel() // t.shape[0]) * \
                    t.element_size()
                t, host = t[early[1]:], host[early[1]:]
                self._early = None
            if host.flags.c_contiguous:
                torch.from_numpy(host).copy_(t, non_blocking=True)
            else:
                host[...] = t.cpu().numpy()
            self.d2h_bytes += t.numel() * t.element_size()
        torch.cuda.synchronize(self.device)


def _sparse_groups(c) -> list:
    """Main statements of a sparse cluster split per target: increments of
    different fields never interact, so each field's 2^d corner statements
    become one stage (per-point order within a field is preserved)."""
    mains = [e for e in c.eqs if e.lhs.func.kind != "temp"]
    if all(e.is_increment for e in mains):
        groups: Dict[str, list] = {}
        for e in mains:
            groups.setdefault(e.lhs.func.name, []).append(e)
        return list(groups.values())
    return [[e] for e in mains]


def _factor_list(e: Expr) -> list:
    return list(e.children) if isinstance(e, Mul) else [e]


def _time_shift(acc: Access) -> int:
    for pos, dim, loop, k in access_offsets(acc):
        if dim.is_time:
            if k is OPAQUE:
                raise BackendError("non-affine time index in %r" % (acc,))
            return k
    raise BackendError("access %r has no time axis" % (acc,))


def _time_varying(e: Expr) -> bool:
    return _dse.time_varying(e)


from .iet import IetNode, build_iet, device_source  # noqa: E402
