"""Seeded synthetic workloads of BASELINE.json's configs.

No public dataset is involved: every input is generated here with the
shapes, units and value ranges BASELINE.json states (h in m, v in km/s,
t/dt in ms, f0 in kHz; origin at the corner of the damping-inclusive grid,
depth = last axis z).

Used by bench.py and the tests; the product package never imports it.
"""

from __future__ import annotations

import math
from typing import Dict, Tuple

import numpy as np

import paper_1807_03032_b200.symbolic as S
from paper_1807_03032_b200.backend.operator import Operator


def ricker(nt: int, dt: float, f0: float) -> np.ndarray:
    t = np.arange(nt) * dt
    a = (math.pi * f0 * (t - 1.0 / f0)) ** 2
    return (1 - 2 * a) * np.exp(-a)


def damping_profile(shape, nbl: int, halo: int, scale: float = 0.1):
    """damp = scale * sum_axes p(delta), p(d) = d - sin(2 pi d)/(2 pi) in the
    nbl outermost layers, 0 inside."""
    nd = len(shape)
    out = np.zeros(tuple(s + 2 * halo for s in shape), np.float64)
    for ax in range(nd):
        prof = np.zeros(shape[ax] + 2 * halo)
        for i in range(nbl):
            d = (nbl - i) / nbl
            v = d - math.sin(2 * math.pi * d) / (2 * math.pi)
            prof[halo + i] = v
            prof[halo + shape[ax] - 1 - i] = v
        sh = [1] * nd
        sh[ax] = -1
        out += prof.reshape(sh)
    return scale * out


def acoustic_operator(shape, h, so, src_coords, rec_coords, dtype="f32",
                      mode="advanced", damp=True, names=("u", "m", "damp")):
    """Reference-API acoustic operator (solve_for of m u_tt - lap u +
    damp u_t) + injection + interpolation."""
    return Operator(acoustic_equations(shape, h, so, src_coords, rec_coords,
                                       damp, names), mode=mode, dtype=dtype)


def acoustic_equations(shape, h, so, src_coords, rec_coords, damp=True,
                       names=("u", "m", "damp"), S=S):
    """The equations of ``acoustic_operator`` built with the symbolic module
    ``S`` (this package's, or the reference's for golden generation)."""
    g = S.Grid(shape, extent=tuple(h * (n - 1) for n in shape))
    u = S.FunctionDecl(names[0], "timefunction", g, space_order=so,
                       time_order=2)
    m = S.FunctionDecl(names[1], "function", g, space_order=so)
    dmp = S.FunctionDecl(names[2], "function", g, space_order=so)
    src = S.FunctionDecl("src", "sparsetimefunction", g,
                         npoint=len(src_coords), coordinates=src_coords)
    pde = m.at * S.dt2(u) - S.laplace(u)
    if damp:
        pde = pde + dmp.at * S.dt(u)
    dt = S.Symbol("dt")
    eqs = [S.Eq(u.forward, S.solve_for(pde, u.forward))]
    eqs += S.inject(src, u.forward, S.mul(src.at, dt, dt, S.pow_(m.at, -1)))
    if len(rec_coords):
        rec = S.FunctionDecl("rec", "sparsetimefunction", g,
                             npoint=len(rec_coords), coordinates=rec_coords)
        eqs += S.interpolate(rec, u.at)
    return eqs


def config1(nt: int = 200, seed: int = 0, dtype: str = "f32",
            src_depth: float = None) -> Tuple[Operator, Dict, float, dict]:
    """Config 1: acoustic so=4, 128^3 interior + 10-point damping (148^3),
    h = 10 m, two-layer velocity (1.5 km/s above the middle depth, a seeded
    U[2.0, 3.0] km/s below), dt = 0.4 h / vmax, 10 Hz Ricker at the grid
    centre, 101 receivers on a line at x = 100 + 12.7 i m, y = 735 m, 20 m
    below the interior top (z = 120 m). ``src_depth`` moves the source (the
    parity variant of SURVEY.md §8d puts it at z = 320 m so the receivers
    record an arrival within nt)."""
    rng = np.random.default_rng(seed)
    h, nbl, so = 10.0, 10, 4
    N = 128 + 2 * nbl
    shape = (N, N, N)
    vlow = float(rng.uniform(2.0, 3.0))
    vz = np.where(np.arange(N) < N // 2, 1.5, vlow)
    dt = 0.4 * h / vlow
    c = h * (N - 1) / 2
    src = [(c, c, c if src_depth is None else src_depth)]
    rec = [(100.0 + 12.7 * i, c, 120.0) for i in range(101)]
    op = acoustic_operator(shape, h, so, src, rec, dtype)
    bufs = op.allocate(nt)
    H = so // 2
    npdt = np.float32 if dtype == "f32" else np.float64
    mz = np.zeros(N + 2 * H)
    mz[H:H + N] = 1.0 / vz ** 2
    mz[:H], mz[H + N:] = mz[H], mz[H + N - 1]
    bufs["m"].data[...] = mz.astype(npdt)[None, None, :]
    bufs["damp"].data[...] = damping_profile(shape, nbl, H).astype(npdt)
    bufs["src"].data[:, 0] = ricker(nt, dt, 0.010).astype(npdt)
    meta = {"shape": shape, "so": so, "nt": nt, "dt": dt, "h": h,
            "nrec": len(rec), "vmax": vlow, "l2_resident": True,
            "src_coords": src, "rec_coords": rec}
    return op, bufs, dt, meta


def config2(so: int = 8, n: int = 512, nbl: int = 40, nt: int = 500,
            nrec_side: int = 512, seed: int = 0, dtype: str = "f32",
            x_planes: int = None) -> Tuple[Operator, Dict, float, dict]:
    """Config 2: acoustic so in {8,12,16}, n^3 interior + nbl damping,
    h = 20 m, seeded 8-layer velocity (sorted U[1.5, 4.5] km/s, random
    interface depths), CFL dt, 15 Hz Ricker 20 m below the interior top at
    the x-y centre, nrec_side^2 receivers on the interior x-y nodes 10 m
    below the interior top. ``x_planes`` keeps only that many x planes
    (bounded CPU-baseline samples of the same per-point work)."""
    rng = np.random.default_rng(seed)
    h = 20.0
    N = n + 2 * nbl
    nx = N if x_planes is None else x_planes
    shape = (nx, N, N)
    vel = np.sort(rng.uniform(1.5, 4.5, 8))
    cuts = nbl + np.sort(rng.choice(np.arange(1, n), 7, replace=False))
    vz = np.empty(N)
    edges = [0] + list(cuts) + [N]
    for k in range(8):
        vz[edges[k]:edges[k + 1]] = vel[k]
    vmax = float(vel.max())
    dt = 0.4 * h / vmax
    xc = h * (nx - 1) / 2
    yc = h * (N - 1) / 2
    src = [(xc, yc, nbl * h + 20.0)]
    ii = np.arange(nrec_side)
    xs = (nbl + ii) * h if x_planes is None else \
        np.linspace(0.0, h * (nx - 1), nrec_side)
    ys = (nbl + ii) * h
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    rec = np.stack([gx.ravel(), gy.ravel(),
                    np.full(gx.size, nbl * h + 10.0)], axis=1)
    rec_list = [tuple(r) for r in rec]
    op = acoustic_operator(shape, h, so, src, rec_list, dtype)
    bufs = op.allocate(nt)
    H = so // 2
    npdt = np.float32 if dtype == "f32" else np.float64
    mz = np.zeros(N + 2 * H)
    mz[H:H + N] = 1.0 / vz ** 2
    mz[:H], mz[H + N:] = mz[H], mz[H + N - 1]
    bufs["m"].data[...] = mz.astype(npdt)[None, None, :]
    dshape = (nx, N, N)
    bufs["damp"].data[...] = damping_profile(dshape, nbl, H).astype(npdt) \
        if x_planes is None else \
        damping_profile((N, N, N), nbl, H)[:nx + 2 * H].astype(npdt)
    bufs["src"].data[:, 0] = ricker(nt, dt, 0.015).astype(npdt)
    meta = {"shape": shape, "so": so, "nt": nt, "dt": dt, "h": h,
            "nrec": rec.shape[0], "vmax": vmax, "src_coords": src,
            "rec_coords": rec_list}
    return op, bufs, dt, meta


def seed_interior(bufs, so, seed=3, fields=("u",)):
    """Random U[-1, 1] interiors of the first two time slots (every point
    carries signal from step 0): the config-size parity cases."""
    H = so // 2
    rng = np.random.default_rng(seed)
    for k in fields:
        inner = bufs[k].data[0:2, H:-H, H:-H, H:-H]
        inner[...] = rng.uniform(-1, 1, inner.shape).astype(inner.dtype)


def smoothed_field(rng, shape, lo, hi, sigma=5.0, dtype=np.float32):
    """Seeded U[0,1] noise, separable Gaussian (sigma in points), min-max
    rescaled to [lo, hi]."""
    from scipy.ndimage import gaussian_filter
    a = gaussian_filter(rng.uniform(0, 1, shape).astype(np.float32), sigma,
                        mode="nearest")
    a = (a - a.min()) / max(float(a.max() - a.min()), 1e-30)
    return (lo + (hi - lo) * a).astype(dtype)


def tti_operator(shape, h, so, src_coords, rec_coords=None, dtype="f32"):
    from paper_1807_03032_b200.operators import tti_equations
    g = S.Grid(shape, extent=tuple(h * (n - 1) for n in shape))
    p = S.FunctionDecl("p", "timefunction", g, space_order=so)
    r = S.FunctionDecl("r", "timefunction", g, space_order=so)
    f = {n: S.FunctionDecl(n, "function", g, space_order=so)
         for n in ("m", "damp", "epsilon", "delta", "theta", "phi")}
    src = S.FunctionDecl("src", "sparsetimefunction", g,
                         npoint=len(src_coords), coordinates=src_coords)
    eqs = tti_equations(p, r, f["m"], f["damp"], f["epsilon"], f["delta"],
                        f["theta"], f["phi"])
    dt = S.Symbol("dt")
    expr = S.mul(src.at, dt, dt, S.pow_(f["m"].at, -1))
    eqs += S.inject(src, p.forward, expr) + S.inject(src, r.forward, expr)
    if rec_coords:
        rec = S.FunctionDecl("rec", "sparsetimefunction", g,
                             npoint=len(rec_coords), coordinates=rec_coords)
        eqs += S.interpolate(rec, p.at)
    return Operator(eqs, mode="advanced", dtype=dtype)


def config3(so: int = 12, n: int = 512, nbl: int = 40, nt: int = 500,
            seed: int = 0, dtype: str = "f32"):
    """Config 3: TTI pseudo-acoustic, n^3 + nbl damping, h = 20 m; velocity
    two-layer as config 1 (1.5 km/s upper half, U[2, 3] lower); eps in
    [0, 0.3], delta in [0, 0.2], theta in [0, pi/4], phi in [0, pi/2], each
    Gaussian-smoothed (sigma = 5 points); 15 Hz Ricker at the x-y centre 20 m
    below the interior top; dt = 0.4 h / (vmax sqrt(1 + 2 eps_max))."""
    rng = np.random.default_rng(seed)
    h = 20.0
    N = n + 2 * nbl
    shape = (N, N, N)
    vlow = float(rng.uniform(2.0, 3.0))
    c = h * (N - 1) / 2
    op = tti_operator(shape, h, so, [(c, c, nbl * h + 20.0)], dtype=dtype)
    bufs = op.allocate(nt)
    H = so // 2
    npdt = np.float32 if dtype == "f32" else np.float64
    st = (N + 2 * H,) * 3
    vz = np.where(np.arange(N + 2 * H) - H < N // 2, 1.5, vlow)
    bufs["m"].data[...] = (1.0 / vz ** 2).astype(npdt)[None, None, :]
    bufs["damp"].data[...] = damping_profile(shape, nbl, H).astype(npdt)
    eps = smoothed_field(rng, st, 0.0, 0.3, dtype=npdt)
    bufs["epsilon"].data[...] = eps
    bufs["delta"].data[...] = smoothed_field(rng, st, 0.0, 0.2, dtype=npdt)
    bufs["theta"].data[...] = smoothed_field(rng, st, 0.0, math.pi / 4,
                                             dtype=npdt)
    bufs["phi"].data[...] = smoothed_field(rng, st, 0.0, math.pi / 2,
                                           dtype=npdt)
    dt = 0.4 * h / (max(1.5, vlow) * math.sqrt(1 + 2 * float(eps.max())))
    bufs["src"].data[:, 0] = ricker(nt, dt, 0.015).astype(npdt)
    meta = {"shape": shape, "so": so, "nt": nt, "dt": dt, "h": h, "nrec": 0,
            "vmax": max(1.5, vlow)}
    return op, bufs, dt, meta


def weak_slab_problem(world: int, rank: int, so: int = 8, n: int = 512,
                      nbl: int = 40, nt: int = 500, nrec_side: int = 512,
                      seed: int = 0, dtype: str = "f32"):
    """Config 2 weak-scaled along x in the config-4 layout: the global grid
    stacks ``world`` config-2 slabs in x ((n + 2 nbl) * world planes, damping
    only at the global ends), one Ricker source per slab, receivers on the
    interior x-y nodes 10 m below the interior top (nrec_side per slab in x).
    Dense buffers are allocated for THIS rank's storage window only (slab +
    so/2 ghost planes per side); sparse buffers are global."""
    from paper_1807_03032_b200.backend.slab import slab_bounds
    rng = np.random.default_rng(seed)
    h = 20.0
    N = n + 2 * nbl
    NX = N * world
    vel = np.sort(rng.uniform(1.5, 4.5, 8))
    cuts = nbl + np.sort(rng.choice(np.arange(1, n), 7, replace=False))
    vz = np.empty(N)
    edges = [0] + list(cuts) + [N]
    for k in range(8):
        vz[edges[k]:edges[k + 1]] = vel[k]
    vmax = float(vel.max())
    dt = 0.4 * h / vmax
    yc = h * (N - 1) / 2
    src = [((s + 0.5) * N * h - 0.5 * h, yc, nbl * h + 20.0)
           for s in range(world)]
    xs = (nbl + np.arange(nrec_side * world)) * h
    ys = (nbl + np.arange(nrec_side)) * h
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    rec = np.stack([gx.ravel(), gy.ravel(),
                    np.full(gx.size, nbl * h + 10.0)], axis=1)
    op = acoustic_operator((NX, N, N), h, so, src, rec, dtype)
    H = so // 2
    a, b = slab_bounds(0, NX - 1, world, H)[rank]
    nw = b - a + 2 * H
    npdt = np.float32 if dtype == "f32" else np.float64
    from paper_1807_03032_b200.backend.operator import _pinned_zeros
    from paper_1807_03032_b200.backend.buffers import DataBuffer
    pin = _pinned_zeros if _cuda() else \
        (lambda shp, dt_: np.zeros(shp, npdt))
    bufs = {}
    for f in op.functions.values():
        if f.kind in ("function", "timefunction"):
            ext = list(f.storage_extents())
            ext[1 if f.kind == "timefunction" else 0] = nw
        else:
            ext = f.storage_extents(nt)
        bufs[f.name] = DataBuffer(f.name, dtype, tuple(ext),
                                  data=pin(tuple(ext), dtype))
    bufs["src_coords"].data[:] = op.functions["src"].coordinate_array
    bufs["rec_coords"].data[:] = op.functions["rec"].coordinate_array
    mz = np.zeros(N + 2 * H)
    mz[H:H + N] = 1.0 / vz ** 2
    mz[:H], mz[H + N:] = mz[H], mz[H + N - 1]
    bufs["m"].data[...] = mz.astype(npdt)[None, None, :]
    # damping over the global grid, sliced to the window (storage planes a..)
    prof_x = np.zeros(NX + 2 * H)
    prof_yz = np.zeros(N + 2 * H)
    for i in range(nbl):
        d = (nbl - i) / nbl
        v = d - math.sin(2 * math.pi * d) / (2 * math.pi)
        prof_x[H + i] = prof_x[H + NX - 1 - i] = v
        prof_yz[H + i] = prof_yz[H + N - 1 - i] = v
    px = prof_x[a:a + nw]
    bufs["damp"].data[...] = (0.1 * (px[:, None, None] + prof_yz[None, :, None]
                                     + prof_yz[None, None, :])).astype(npdt)
    w = ricker(nt, dt, 0.015).astype(npdt)
    bufs["src"].data[:] = w[:, None]
    meta = {"shape": (NX, N, N), "so": so, "nt": nt, "dt": dt, "h": h,
            "nrec": rec.shape[0], "slab": (a, b)}
    return op, bufs, dt, meta


def tti_weak_slab(world: int, rank: int, so: int = 12, n: int = 512,
                  nbl: int = 40, nt: int = 500, seed: int = 0,
                  dtype: str = "f32"):
    """Config 3 weak-scaled along x: ``world`` copies of the config-3 cube
    stacked in x (damping at the global x ends and on every y/z face), the
    anisotropy fields of one cube repeated per slab (so every rank's ghost
    planes hold exactly its neighbour's values), one Ricker source per
    slab. Dense buffers hold THIS rank's storage window only."""
    from paper_1807_03032_b200.backend.slab import slab_bounds
    from paper_1807_03032_b200.backend.operator import _pinned_zeros
    from paper_1807_03032_b200.backend.buffers import DataBuffer
    rng = np.random.default_rng(seed)
    h = 20.0
    N = n + 2 * nbl
    NX = N * world
    H = so // 2
    vlow = float(rng.uniform(2.0, 3.0))
    c = h * (N - 1) / 2
    src = [((s + 0.5) * N * h - 0.5 * h, c, nbl * h + 20.0)
           for s in range(world)]
    op = tti_operator((NX, N, N), h, so, src, dtype=dtype)
    a, b = slab_bounds(0, NX - 1, world, H)[rank]
    nw = b - a + 2 * H
    npdt = np.float32 if dtype == "f32" else np.float64
    pin = _pinned_zeros if _cuda() else (lambda shp, dt_: np.zeros(shp, npdt))
    bufs = {}
    for f in op.functions.values():
        if f.kind in ("function", "timefunction"):
            ext = list(f.storage_extents())
            ext[1 if f.kind == "timefunction" else 0] = nw
        else:
            ext = f.storage_extents(nt)
        bufs[f.name] = DataBuffer(f.name, dtype, tuple(ext),
                                  data=pin(tuple(ext), dtype))
    bufs["src_coords"].data[:] = op.functions["src"].coordinate_array
    # storage plane x of the global grid -> plane of the one-cube field
    xs = np.arange(a, a + nw)
    inner = (xs >= H) & (xs < NX + H)
    cube_x = np.where(inner, H + (xs - H) % N,
                      np.where(xs < H, xs, xs - N * (world - 1)))
    st = (N + 2 * H,) * 3
    vz = np.where(np.arange(N + 2 * H) - H < N // 2, 1.5, vlow)
    bufs["m"].data[...] = (1.0 / vz ** 2).astype(npdt)[None, None, :]
    eps_max = 0.0
    for name, lo, hi in (("epsilon", 0.0, 0.3), ("delta", 0.0, 0.2),
                         ("theta", 0.0, math.pi / 4),
                         ("phi", 0.0, math.pi / 2)):
        fld = smoothed_field(rng, st, lo, hi, dtype=npdt)
        bufs[name].data[...] = fld[cube_x]
        if name == "epsilon":
            eps_max = float(fld.max())
        del fld
    prof_x = np.zeros(NX + 2 * H)
    prof_yz = np.zeros(N + 2 * H)
    for i in range(nbl):
        d = (nbl - i) / nbl
        v = d - math.sin(2 * math.pi * d) / (2 * math.pi)
        prof_x[H + i] = prof_x[H + NX - 1 - i] = v
        prof_yz[H + i] = prof_yz[H + N - 1 - i] = v
    px = prof_x[a:a + nw]
    bufs["damp"].data[...] = (0.1 * (px[:, None, None] + prof_yz[None, :, None]
                                     + prof_yz[None, None, :])).astype(npdt)
    dt = 0.4 * h / (max(1.5, vlow) * math.sqrt(1 + 2 * eps_max))
    bufs["src"].data[:] = ricker(nt, dt, 0.015).astype(npdt)[:, None]
    meta = {"shape": (NX, N, N), "so": so, "nt": nt, "dt": dt, "h": h,
            "nrec": 0, "slab": (a, b)}
    return op, bufs, dt, meta


def _smoothed_window_gpu(seed: int, nx: int, ny: int, nz: int, x0: int,
                         x1: int, lo: float, hi: float, sigma: float = 5.0):
    """Planes [x0, x1) of a field of shape (nx, ny, nz): per-plane seeded
    U[0,1] noise (any rank regenerates any plane), separable Gaussian
    (sigma points, radius 4 sigma, edge-replicating at the global
    boundary), rescaled to [lo, hi] with the analytic spread of smoothed
    uniform noise (1/2 +- 5 std, clipped) so that every rank maps values
    identically without a global min/max. Runs on the current GPU;
    returns a host float32 array."""
    import torch
    import torch.nn.functional as F
    rad = int(4 * sigma + 0.5)
    a, b = max(x0 - rad, 0), min(x1 + rad, nx)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    vol = torch.empty((b - a, ny, nz), device=dev, dtype=torch.float32)
    for x in range(a, b):
        g.manual_seed(seed * 1000003 + x)
        vol[x - a] = torch.rand((ny, nz), generator=g, device=dev)
    k = torch.arange(-rad, rad + 1, device=dev, dtype=torch.float32)
    w = torch.exp(-0.5 * (k / sigma) ** 2)
    w = (w / w.sum()).view(1, 1, -1)
    std = math.sqrt(1.0 / 12.0) * float((w ** 2).sum().sqrt()) ** 3

    def conv(v, axis, pad_lo, pad_hi):
        v = v.movedim(axis, -1).contiguous()
        shp = v.shape
        flat = F.pad(v.view(-1, 1, shp[-1]), (pad_lo, pad_hi), mode="replicate")
        del v
        out = F.conv1d(flat, w)
        del flat
        return out.view(*shp[:-1], out.shape[-1]).movedim(-1, axis)

    vol = conv(vol, 2, rad, rad)
    vol = conv(vol, 1, rad, rad)
    # x: real neighbouring planes inside the grid, replicated beyond it
    vol = conv(vol, 0, rad - (x0 - a), rad - (b - x1))
    vol = ((vol - 0.5) / (10.0 * std) + 0.5).clamp_(0.0, 1.0)
    host = (lo + (hi - lo) * vol).cpu().numpy()
    del vol
    torch.cuda.empty_cache()
    return host


def config5_slab(world: int, rank: int, so: int = 12, nt: int = 300,
                 n: tuple = (1536, 1024, 1024), nbl: int = 40,
                 nrec: tuple = (1024, 1024), dtype: str = "f32"):
    """Config 5 (TTI strong scaling): (1536 x 1024 x 1024) interior + 40-point
    damping = 1616 x 1104 x 1104, so=12, h = 20 m, two-layer velocity as
    config 1, eps/delta/theta/phi Gaussian-smoothed (sigma = 5 points) from
    per-plane seeded noise (generated on the GPU for THIS rank's window, so
    every rank sees the same global field), 15 Hz Ricker 20 m below the
    interior top at the x-y centre, 1024 x 1024 receivers 10 m below it on
    the central interior x nodes and all interior y nodes, nt = 300. Dense
    buffers hold this rank's storage window only."""
    from paper_1807_03032_b200.backend.slab import slab_bounds
    from paper_1807_03032_b200.backend.operator import _pinned_zeros
    from paper_1807_03032_b200.backend.buffers import DataBuffer
    rng = np.random.default_rng(5)
    h = 20.0
    NX, NY, NZ = (m + 2 * nbl for m in n)
    H = so // 2
    vlow = float(rng.uniform(2.0, 3.0))
    xc, yc = h * (NX - 1) / 2, h * (NY - 1) / 2
    xr = (nbl + (n[0] - nrec[0]) // 2 + np.arange(nrec[0])) * h
    yr = (nbl + np.arange(nrec[1])) * h
    gx, gy = np.meshgrid(xr, yr, indexing="ij")
    rec = np.stack([gx.ravel(), gy.ravel(),
                    np.full(gx.size, nbl * h + 10.0)], axis=1)
    op = tti_operator((NX, NY, NZ), h, so, [(xc, yc, nbl * h + 20.0)],
                      rec_coords=[tuple(r) for r in rec], dtype=dtype)
    a, b = slab_bounds(0, NX - 1, world, H)[rank]
    nw = b - a + 2 * H
    npdt = np.float32
    bufs = {}
    for f in op.functions.values():
        if f.kind in ("function", "timefunction"):
            ext = list(f.storage_extents())
            ext[1 if f.kind == "timefunction" else 0] = nw
        else:
            ext = f.storage_extents(nt)
        bufs[f.name] = DataBuffer(f.name, dtype, tuple(ext),
                                  data=_pinned_zeros(tuple(ext), dtype))
    bufs["src_coords"].data[:] = op.functions["src"].coordinate_array
    bufs["rec_coords"].data[:] = op.functions["rec"].coordinate_array
    st = (NX + 2 * H, NY + 2 * H, NZ + 2 * H)
    vz = np.where(np.arange(NZ + 2 * H) - H < NZ // 2, 1.5, vlow)
    bufs["m"].data[...] = (1.0 / vz ** 2).astype(npdt)[None, None, :]
    for i, (name, lo, hi) in enumerate((("epsilon", 0.0, 0.3),
                                        ("delta", 0.0, 0.2),
                                        ("theta", 0.0, math.pi / 4),
                                        ("phi", 0.0, math.pi / 2))):
        bufs[name].data[...] = _smoothed_window_gpu(
            1000 + i, st[0], st[1], st[2], a, a + nw, lo, hi)
    prof = [np.zeros(s_) for s_ in st]
    for i in range(nbl):
        d = (nbl - i) / nbl
        v = d - math.sin(2 * math.pi * d) / (2 * math.pi)
        for ax, N in enumerate((NX, NY, NZ)):
            prof[ax][H + i] = prof[ax][H + N - 1 - i] = v
    for i, v in enumerate(prof[0][a:a + nw]):   # plane by plane: no 16 GB temp
        bufs["damp"].data[i] = (0.1 * ((v + prof[1][:, None])
                                       + prof[2][None, :])).astype(npdt)
    dt = 0.4 * h / (max(1.5, vlow) * math.sqrt(1 + 2 * 0.3))
    bufs["src"].data[:, 0] = ricker(nt, dt, 0.015).astype(npdt)
    meta = {"shape": (NX, NY, NZ), "so": so, "nt": nt, "dt": dt, "h": h,
            "nrec": rec.shape[0], "slab": (a, b)}
    return op, bufs, dt, meta


def config4_slab(world: int, rank: int, so: int = 8, n: int = 1024,
                 nt: int = 200, dtype: str = "f32"):
    """Config 4 (weak scaling): acoustic so=8, an n^3 interior per GPU
    stacked along x ((n * world) x n x n, no damping layer: the damp field
    is kept, all zero, so the bytes per point are unchanged), h = 10 m,
    two-layer velocity as config 1, one 10 Hz Ricker at the centre of each
    slab, no receivers, nt = 200. Dense buffers hold THIS rank's storage
    window only (slab + so/2 ghost planes per side)."""
    from paper_1807_03032_b200.backend.slab import slab_bounds
    from paper_1807_03032_b200.backend.operator import _pinned_zeros
    from paper_1807_03032_b200.backend.buffers import DataBuffer
    rng = np.random.default_rng(0)
    h = 10.0
    NX = n * world
    vlow = float(rng.uniform(2.0, 3.0))
    vz = np.where(np.arange(n) < n // 2, 1.5, vlow)
    dt = 0.4 * h / vlow
    c = h * (n - 1) / 2
    src = [((s + 0.5) * n * h - 0.5 * h, c, c) for s in range(world)]
    op = acoustic_operator((NX, n, n), h, so, src, [], dtype)
    H = so // 2
    a, b = slab_bounds(0, NX - 1, world, H)[rank]
    nw = b - a + 2 * H
    npdt = np.float32 if dtype == "f32" else np.float64
    pin = _pinned_zeros if _cuda() else (lambda shp, dt_: np.zeros(shp, npdt))
    bufs = {}
    for f in op.functions.values():
        if f.kind in ("function", "timefunction"):
            ext = list(f.storage_extents())
            ext[1 if f.kind == "timefunction" else 0] = nw
        else:
            ext = f.storage_extents(nt)
        bufs[f.name] = DataBuffer(f.name, dtype, tuple(ext),
                                  data=pin(tuple(ext), dtype))
    bufs["src_coords"].data[:] = op.functions["src"].coordinate_array
    mz = np.zeros(n + 2 * H)
    mz[H:H + n] = 1.0 / vz ** 2
    mz[:H], mz[H + n:] = mz[H], mz[H + n - 1]
    bufs["m"].data[...] = mz.astype(npdt)[None, None, :]
    bufs["src"].data[:] = ricker(nt, dt, 0.010).astype(npdt)[:, None]
    meta = {"shape": (NX, n, n), "so": so, "nt": nt, "dt": dt, "h": h,
            "nrec": 0, "slab": (a, b)}
    return op, bufs, dt, meta


def _cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
