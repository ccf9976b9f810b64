"""Front end restated from the reference (symbolic/): known answers mirroring
the reference's own unit tests (tests/test_fd.py, test_sparse.py,
test_backend.py error conventions)."""

from fractions import Fraction

import pytest

from paper_1807_03032_b200.symbolic import (Constant, DeclarationError, Eq,
                                            FunctionDecl, Grid, SolveError,
                                            centered_weights, derivative,
                                            dt2, evaluate, fornberg_weights,
                                            inject, interpolate, laplace,
                                            num, solve_for)
from paper_1807_03032_b200.symbolic.expr import Add, Mul, add, mul


def test_fornberg_exact():
    assert fornberg_weights(1, (-1, 0, 1)) == [Fraction(-1, 2), 0, Fraction(1, 2)]
    assert fornberg_weights(2, (-1, 0, 1)) == [1, -2, 1]
    w = centered_weights(4, 2)
    assert w == {-2: Fraction(-1, 12), -1: Fraction(4, 3), 0: Fraction(-5, 2),
                 1: Fraction(4, 3), 2: Fraction(-1, 12)}
    w8 = centered_weights(8, 2)
    assert w8[0] == Fraction(-205, 72) and w8[4] == Fraction(-1, 560)


@pytest.mark.parametrize("order,deriv", [(2, 1), (4, 1), (4, 2), (8, 2), (16, 2)])
def test_weights_exact_on_monomials(order, deriv):
    w = centered_weights(order, deriv)
    for k in range(order + 1):
        s = sum(c * Fraction(o) ** k for o, c in w.items())
        want = 0
        if k == deriv:
            want = 1
            for i in range(2, deriv + 1):
                want *= i
        assert s == want


def test_canonical_forms():
    g = Grid((5,))
    u = FunctionDecl("u", "timefunction", g, space_order=2)
    a = u.at
    assert add(a, a) == mul(num(2), a)
    assert isinstance(add(a, num(1)), Add)
    assert mul(a, num(0)) == Constant(Fraction(0))
    assert isinstance(mul(a, a), type(a ** 2))


def test_solve_wave_equation():
    g = Grid((11,), extent=(10.0,))
    u = FunctionDecl("u", "timefunction", g, space_order=2)
    m = FunctionDecl("m", "function", g, space_order=2)
    sol = solve_for(m.at * dt2(u) - laplace(u), u.forward)
    vals = {"u_f": 0.0, "u": 1.0, "u_b": 0.5, "um": 0.25, "up": 0.75,
            "m": 2.0}
    env = {"dt": 0.1, "h_x": 1.0, "t": 0.0, "x": 3.0}

    def acc(a):
        t = evaluate(a.indices[0], env)
        x = evaluate(a.indices[1], env) if len(a.indices) > 1 else 0
        if a.func.name == "m":
            return 2.0
        if t == 0.0:
            return {2.0: 0.25, 3.0: 1.0, 4.0: 0.75}[x]
        return 0.5
    got = evaluate(sol, env, on_access=acc)
    lap = 0.25 - 2 * 1.0 + 0.75
    want = 2 * 1.0 - 0.5 + 0.1 ** 2 * lap / 2.0
    assert got == pytest.approx(want, rel=1e-12)


def test_solve_errors():
    g = Grid((5,))
    u = FunctionDecl("u", "timefunction", g)
    with pytest.raises(SolveError):
        solve_for(u.at * u.forward * u.forward, u.forward)
    with pytest.raises(SolveError):
        solve_for(u.at, u.forward)


def test_declaration_errors():
    with pytest.raises(DeclarationError):
        Grid((1, 4))
    g = Grid((11,), extent=(10.0,))
    with pytest.raises(DeclarationError):
        FunctionDecl("u", "timefunction", g, space_order=3)
    with pytest.raises(DeclarationError):
        FunctionDecl("q", "sparsetimefunction", g, npoint=1,
                     coordinates=[(11.5,)])
    FunctionDecl("q", "sparsetimefunction", g, npoint=1, coordinates=[(10.0,)])


def _weights(eqs, coord):
    env = {"h_x": 1.0, "o_x": 0.0, "t": 0.0, "p_q": 0.0, "dt": 1.0}

    def acc(a):
        return coord if a.func.kind == "coordinates" else 1.0
    return [evaluate(eq.rhs, env, on_access=acc) for eq in eqs]


def test_inject_weights():
    g = Grid((11,), extent=(10.0,))
    u = FunctionDecl("u", "timefunction", g, space_order=2)
    q = FunctionDecl("q", "sparsetimefunction", g, npoint=1,
                     coordinates=[(4.0,)])
    assert _weights(inject(q, u.forward, num(1)), 4.0) == [1.0, 0.0]
    assert _weights(inject(q, u.forward, num(1)), 4.5) == [0.5, 0.5]


def test_interpolate_partition_of_unity():
    g = Grid((11, 11), extent=(10.0, 10.0))
    u = FunctionDecl("u", "timefunction", g, space_order=2)
    rec = FunctionDecl("rec", "sparsetimefunction", g, npoint=1,
                       coordinates=[(3.3, 7.1)])
    eq = interpolate(rec, u.at)[0]
    env = {"h_x": 1.0, "h_y": 1.0, "o_x": 0.0, "o_y": 0.0, "t": 0.0,
           "p_rec": 0.0}

    def acc(a):
        if a.func.kind == "coordinates":
            return rec.coordinate_values[0][int(a.indices[1].value)]
        return 3.0
    assert evaluate(eq.rhs, env, on_access=acc) == pytest.approx(3.0)
