"""Canonical operator constructions with the reference API.

``tti_equations`` authors the pseudo-acoustic TTI system the reference does
not ship with the reference's own
primitives (``derivative``/``derivative_of``, ``solve_for``, builtin calls):

    m p_tt + damp p_t = (1 + 2 eps) H_xy(p) + sqrt(1 + 2 delta) H_z(r)
    m r_tt + damp r_t = sqrt(1 + 2 delta) H_xy(p) + H_z(r)

with a = (sin th cos ph, sin th sin ph, cos th), H_z(f) = a.grad(a.grad f)
(first derivatives of order so/2 nested, so the reach equals the so/2 halo;
full-order nesting would read past the halo) and
H_xy(p) = lap_so(p) - H_z(p). ``S`` is the symbolic module (this package's
or the reference's), so the oracle and the backend build identical trees.

``acoustic_equation`` is the isotropic update (solve_for of
m u_tt - lap u [+ damp u_t]) for completeness.
"""

from __future__ import annotations


def _S(S):
    if S is None:
        from . import symbolic as S
    return S


def acoustic_equation(u, m, damp=None, S=None):
    S = _S(S)
    pde = m.at * S.dt2(u) - S.laplace(u)
    if damp is not None:
        pde = pde + damp.at * S.dt(u)
    return S.Eq(u.forward, S.solve_for(pde, u.forward))


def tti_direction(theta, phi, S=None):
    S = _S(S)
    st, ct = S.call("sin", theta.at), S.call("cos", theta.at)
    sp, cp = S.call("sin", phi.at), S.call("cos", phi.at)
    return [S.mul(st, cp), S.mul(st, sp), ct]


def rotated_hz(f, a, S=None):
    """H_z(f) = sum_i a_i d_i (sum_j a_j d_j f), inner/outer order so/2."""
    S = _S(S)
    g = f.grid
    so = f.space_order
    dims = g.dimensions
    inner = S.add(*[S.mul(a[j], S.derivative(f, dims[j], so // 2, 1))
                    for j in range(g.ndim)])
    return S.add(*[S.mul(a[i], S.derivative_of(inner, dims[i], so // 2, 1,
                                               g.spacing_of(dims[i])))
                   for i in range(g.ndim)])


def tti_equations(p, r, m, damp, eps, delta, theta, phi, S=None):
    S = _S(S)
    a = tti_direction(theta, phi, S)
    hzp = rotated_hz(p, a, S)
    hzr = rotated_hz(r, a, S)
    hxy = S.laplace(p) - hzp
    e2 = 1 + 2 * eps.at
    sd = S.call("sqrt", 1 + 2 * delta.at)
    pde_p = m.at * S.dt2(p) + damp.at * S.dt(p) - (e2 * hxy + sd * hzr)
    pde_r = m.at * S.dt2(r) + damp.at * S.dt(r) - (sd * hxy + hzr)
    return [S.Eq(p.forward, S.solve_for(pde_p, p.forward)),
            S.Eq(r.forward, S.solve_for(pde_r, r.forward))]
