"""Seeded parity cases shared by make_golden.py (runs the real reference in
the build container) and the tests (run the oracle port / the GPU path).

``build(S, case)`` takes a symbolic module -- the reference's
``stencilc.symbolic`` or ours -- so both sides construct identical equations;
``fill(bufs, case)`` writes identical seeded inputs into either side's
buffers. Inputs mimic SURVEY.md §8(d): layered velocity, damping layer,
Ricker source, off-node sources/receivers (plus on-node and upper-extent
points), optional random initial wavefields so every grid point carries
signal from step 0.
"""

from __future__ import annotations

import math

import numpy as np

# name, ndim, N, so, dtype, mode, damp, nt, nrec, random_init
CASES = [
    ("ac3d_so4_f32_adv", 3, 24, 4, "f32", "advanced", True, 20, 16, True),
    ("ac3d_so8_f32_adv", 3, 24, 8, "f32", "advanced", True, 20, 16, True),
    ("ac3d_so12_f32_adv", 3, 28, 12, "f32", "advanced", True, 12, 8, True),
    ("ac3d_so16_f32_adv", 3, 32, 16, "f32", "advanced", True, 10, 8, True),
    ("ac3d_so2_f32_adv", 3, 20, 2, "f32", "advanced", True, 20, 8, True),
    ("ac3d_so8_f32_basic", 3, 24, 8, "f32", "basic", True, 16, 16, True),
    ("ac3d_so8_f32_aggr", 3, 24, 8, "f32", "aggressive", True, 16, 8, True),
    ("ac3d_so4_f32_nodamp", 3, 24, 4, "f32", "advanced", False, 20, 16, False),
    ("ac3d_so8_f64_adv", 3, 24, 8, "f64", "advanced", True, 16, 16, True),
    ("ac3d_so4_f64_basic", 3, 20, 4, "f64", "basic", False, 16, 8, True),
    ("ac2d_so4_f32_adv", 2, 40, 4, "f32", "advanced", True, 30, 8, True),
    ("ac1d_so4_f32_adv", 1, 64, 4, "f32", "advanced", True, 40, 4, True),
    ("ac2d_so8_f64_basic", 2, 36, 8, "f64", "basic", True, 20, 8, True),
    ("ac3d_so8_f32_src4", 3, 24, 8, "f32", "advanced", True, 16, 16, False),
]

FIELDS = ("u", "rec")


def case_dict(row):
    keys = ("name", "ndim", "N", "so", "dtype", "mode", "damp", "nt", "nrec",
            "rand")
    return dict(zip(keys, row))


def geometry(case):
    nd, N = case["ndim"], case["N"]
    h = 10.0
    ext = h * (N - 1)
    rng = np.random.default_rng(1234 + nd * 100 + N)
    nsrc = 4 if case["name"].endswith("src4") else 1
    centre = ext / 2
    src = [tuple(centre + [3.3, -1.7, 2.1][d] for d in range(nd))]
    for k in range(1, nsrc):
        src.append(tuple(centre + 12.5 * k * (d + 1) * 0.3 for d in range(nd)))
    recs = []
    nrec = case["nrec"]
    for i in range(nrec):
        if i == 0:
            recs.append(tuple(ext for _ in range(nd)))      # upper extent
        elif i == 1:
            recs.append(tuple(h * 3 for _ in range(nd)))    # on a node
        elif i == 2:
            recs.append(tuple([33.3, 55.0, 20.0][d] for d in range(nd)))
        else:
            recs.append(tuple(float(x) for x in rng.uniform(0, ext, nd)))
    return h, ext, src, recs


def build(S, case):
    """Equations with the reference API of module ``S``."""
    nd, N, so = case["ndim"], case["N"], case["so"]
    h, ext, src_c, rec_c = geometry(case)
    g = S.Grid((N,) * nd, extent=(ext,) * nd)
    u = S.FunctionDecl("u", "timefunction", g, space_order=so, time_order=2)
    m = S.FunctionDecl("m", "function", g, space_order=so)
    damp = S.FunctionDecl("damp", "function", g, space_order=so)
    src = S.FunctionDecl("src", "sparsetimefunction", g, npoint=len(src_c),
                         coordinates=src_c)
    rec = S.FunctionDecl("rec", "sparsetimefunction", g, npoint=len(rec_c),
                         coordinates=rec_c)
    pde = m.at * S.dt2(u) - S.laplace(u)
    if case["damp"]:
        pde = pde + damp.at * S.dt(u)
    stencil = S.Eq(u.forward, S.solve_for(pde, u.forward))
    dt = S.Symbol("dt")
    eqs = [stencil] + S.inject(src, u.forward,
                               S.mul(src.at, dt, dt, S.pow_(m.at, -1))) + \
        S.interpolate(rec, u.at)
    return eqs


def ricker(nt, dt, f0):
    t = np.arange(nt) * dt
    t0 = 1.0 / f0
    a = (math.pi * f0 * (t - t0)) ** 2
    return (1 - 2 * a) * np.exp(-a)


def dt_of(case):
    h = 10.0
    return 0.4 * h / 3.0


def fill(bufs, case):
    """Seeded inputs, identical for any buffer dict with numpy ``.data``."""
    nd, N, so = case["ndim"], case["N"], case["so"]
    H = so // 2
    rng = np.random.default_rng(99 + N + so + nd)
    npdt = np.float32 if case["dtype"] == "f32" else np.float64
    shp = bufs["m"].data.shape
    zi = np.arange(shp[-1]) - H
    v = np.where(zi < N // 2, 1.5, 2.5).astype(np.float64)
    v = np.broadcast_to(v, shp) + 0.3 * rng.uniform(0, 1, shp)
    bufs["m"].data[...] = (1.0 / v ** 2).astype(npdt)
    nbl = 4
    dmp = np.zeros(shp)
    for ax in range(nd):
        idx = np.arange(shp[ax]) - H
        prof = np.zeros(shp[ax])
        for i in range(nbl):
            d = (nbl - i) / nbl
            val = d - math.sin(2 * math.pi * d) / (2 * math.pi)
            prof[i + H] = val
            prof[N - 1 - i + H] = val
        sh = [1] * nd
        sh[ax] = shp[ax]
        dmp = dmp + prof.reshape(sh)
    if "damp" in bufs:
        bufs["damp"].data[...] = (0.1 * dmp).astype(npdt)
    nt = bufs["src"].data.shape[0]
    w = ricker(nt, dt_of(case), 0.05)
    for p in range(bufs["src"].data.shape[1]):
        bufs["src"].data[:, p] = (w * (1 + 0.1 * p)).astype(npdt)
    if case["rand"]:
        u = bufs["u"].data
        inner = tuple(slice(H, H + N) for _ in range(nd))
        for s in range(2):
            u[(s,) + inner] = rng.uniform(-1, 1, (N,) * nd).astype(npdt)
