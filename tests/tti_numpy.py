"""Float64 numpy restatement of the TTI time step (test infrastructure).

The oracle port evaluates the reference's fully expanded TTI trees; at
space order 12/16 building and running it takes ~15 minutes per case, so
the high-order GPU tests check against this direct restatement of the same
discretisation instead (paper_1807_03032_b200/operators.py: rotated_hz,
tti_equations; weights from symbolic/fd.centered_weights, the Fornberg
weights the reference uses, fd.py:27-66):

    g_f   = sum_j a_j D1_j f          (inner order so/2, at every point the
                                       outer stencil reaches: domain + R)
    Hz(f) = sum_i a_i D1_i g_f        (outer order so/2)
    Hxy   = lap_so(p) - Hz(p)
    m (p+ - 2p + p-)/dt^2 + damp (p+ - p-)/(2 dt) = (1+2e) Hxy + sqrt(1+2d) Hz(r)
    m (r+ - 2r + r-)/dt^2 + damp (r+ - r-)/(2 dt) = sqrt(1+2d) Hxy + Hz(r)

on storage arrays with halo so/2 (zero outside the domain), modulo-3 time
slots, t = 0 .. nt-1 (the same slot walk as Operator.apply).
"""

from __future__ import annotations

import numpy as np

from paper_1807_03032_b200.symbolic.fd import centered_weights


def _d1(f, axis, w, h, lo, hi):
    """First derivative along ``axis`` on storage index range [lo, hi) of
    every axis (weights w[k] for k = 1..R, antisymmetric)."""
    sl = [slice(lo, hi)] * 3
    out = np.zeros(tuple(hi - lo for _ in range(3)))
    for k, c in w.items():
        if k <= 0:
            continue
        a = list(sl)
        b = list(sl)
        a[axis] = slice(lo + k, hi + k)
        b[axis] = slice(lo - k, hi - k)
        out += float(c) * (f[tuple(a)] - f[tuple(b)])
    return out / h


def step(p, pm, r, rm, m, damp, eps, delta, theta, phi, so, h, dt):
    """One TTI update on storage arrays (float64); returns (p+, r+) over
    the whole storage extent (halo left zero)."""
    H, R = so // 2, so // 4
    n = p.shape[0]
    w1 = centered_weights(so // 2, 1)
    w2 = centered_weights(so, 2)
    a = [np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi),
         np.cos(theta)]
    glo, ghi = H - R, n - H + R          # g on the domain widened by R

    def hz(f):
        g = sum(a[j][glo:ghi, glo:ghi, glo:ghi] *
                _d1(f, j, w1, h[j], glo, ghi) for j in range(3))
        gs = np.zeros_like(f)
        gs[glo:ghi, glo:ghi, glo:ghi] = g
        return sum(a[i][H:n - H, H:n - H, H:n - H] *
                   _d1(gs, i, w1, h[i], H, n - H) for i in range(3))

    D = (slice(H, n - H),) * 3
    lap = np.zeros(tuple(n - 2 * H for _ in range(3)))
    for ax in range(3):
        for k, c in w2.items():
            s = [slice(H, n - H)] * 3
            s[ax] = slice(H + k, n - H + k)
            lap += float(c) * p[tuple(s)] / (h[ax] * h[ax])
    hzp, hzr = hz(p), hz(r)
    hxy = lap - hzp
    am = m[D] / (dt * dt)
    ad = damp[D] / (2 * dt)
    e2 = 1 + 2 * eps[D]
    sd = np.sqrt(1 + 2 * delta[D])
    pn = np.zeros_like(p)
    rn = np.zeros_like(r)
    pn[D] = (am * (2 * p[D] - pm[D]) + ad * pm[D] + e2 * hxy + sd * hzr) / (am + ad)
    rn[D] = (am * (2 * r[D] - rm[D]) + ad * rm[D] + sd * hxy + hzr) / (am + ad)
    return pn, rn


def run(bufs, so, h, dt, nt):
    """Apply ``nt`` steps to float64 copies of the DataBuffer dict ``bufs``
    (p, r time functions with 3 slots; m, damp, epsilon, delta, theta,
    phi); returns the final (p, r) slot arrays."""
    P = bufs["p"].data.astype(np.float64)
    Rr = bufs["r"].data.astype(np.float64)
    f = {k: bufs[k].data.astype(np.float64)
         for k in ("m", "damp", "epsilon", "delta", "theta", "phi")}
    for t in range(nt):
        c, pv, nx = t % 3, (t - 1) % 3, (t + 1) % 3
        P[nx], Rr[nx] = step(P[c], P[pv], Rr[c], Rr[pv], f["m"], f["damp"],
                             f["epsilon"], f["delta"], f["theta"], f["phi"],
                             so, h, dt)
    return P, Rr
