"""Snapshot (ConditionalDimension) cases: acoustic
propagation that saves every f-th wavefield into a sub-sampled time
function ``us[t/f] = u`` and accumulates ``img += us * u`` (a guarded
read), authored with the reference API; ``build(S, case)`` works with the
reference's symbolic module or ours."""

import numpy as np

# name, shape, so, factor, steps, dtype, mode
CASES = [
    ("snap2d_so4_f3", (20, 18), 4, 3, 10, "f32", "advanced"),
    ("snap3d_so8_f2", (14, 12, 16), 8, 2, 7, "f32", "advanced"),
    ("snap2d_so2_f4_f64", (16, 15), 2, 4, 9, "f64", "aggressive"),
]


def case_dict(row):
    return dict(zip(("name", "shape", "so", "factor", "steps", "dtype",
                     "mode"), row))


def build(S, case):
    shape, so, f = case["shape"], case["so"], case["factor"]
    g = S.Grid(shape, extent=tuple(10.0 * (n - 1) for n in shape))
    m = S.FunctionDecl("m", "function", g, space_order=so)
    u = S.FunctionDecl("u", "timefunction", g, space_order=so)
    save = (case["steps"] + f - 1) // f
    td = S.Dimension("tus", "conditional", parent=g.time_dim, factor=f)
    us = S.FunctionDecl("us", "timefunction", g, space_order=so, save=save,
                        time_dim=td)
    img = S.FunctionDecl("img", "function", g, space_order=so)
    c = tuple(10.0 * (n - 1) / 2 + 3.3 for n in shape)
    src = S.FunctionDecl("src", "sparsetimefunction", g, npoint=1,
                         coordinates=[c])
    eqs = [S.Eq(u.forward, S.solve_for(m.at * S.dt2(u) - S.laplace(u),
                                       u.forward))]
    eqs += S.inject(src, u.forward, S.mul(src.at, S.Symbol("dt"),
                                          S.Symbol("dt"),
                                          S.pow_(m.at, -1)))
    eqs.append(S.Eq(us.at, u.at))
    eqs.append(S.Eq(img.at, img.at + us.at * u.at))
    return eqs


def fill(bufs, case, seed=3):
    rng = np.random.default_rng(seed)
    npdt = np.float32 if case["dtype"] == "f32" else np.float64
    m = bufs["m"].data
    m[...] = (1.0 / rng.uniform(1.5, 2.5, m.shape) ** 2).astype(npdt)
    nt = bufs["src"].data.shape[0]
    bufs["src"].data[:, 0] = np.sin(0.7 * np.arange(nt) + 0.3).astype(npdt)


DT = 2.0
