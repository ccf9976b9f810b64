"""Spec corpus for the CLI parity tests: problem specs in the reference's
line format (pkg/src/stencilc/cli/parser.py) covering declarations, every
expression form, sparse statements, regions, snapshots and params."""

ACOUSTIC_1D = """\
# 1D acoustic operator
grid shape=(21,)
function m space_order=2
timefunction u space_order=2 time_order=2
sparsetimefunction src npoint=1 coords=((10.0,),)
eq u.forward = solve(m*u.dt2 - u.laplace, u.forward)
src.inject(field=u.forward, expr=src * dt**2 / m)
params steps=10 mode=advanced precision=f64
"""

ACOUSTIC_3D = """\
grid shape=(20, 18, 22) extent=(190.0, 170.0, 210.0)
function m space_order=8
function damp space_order=8
timefunction u space_order=8 time_order=2
sparsetimefunction src npoint=1 coords=((95.0, 83.3, 101.7),)
sparsetimefunction rec npoint=3 coords=((20.0, 30.0, 15.0), (100.5, 60.25, 33.0), (180.0, 160.0, 200.0))
eq u.forward = solve(m*u.dt2 - u.laplace + damp*u.dt, u.forward)
src.inject(field=u.forward, expr=src * dt**2 / m)
rec.interpolate(u)
params steps=6 mode=advanced precision=f32
"""

SNAPSHOT_2D = """\
grid shape=(16, 15)
function m space_order=4
timefunction u space_order=4 time_order=2
timefunction us space_order=4 save=4 factor=3
sparsetimefunction src npoint=1 coords=((7.3, 6.1),)
eq u.forward = solve(m*u.dt2 - u.laplace, u.forward)
src.inject(field=u.forward, expr=src * dt**2 / m)
eq us = u
params steps=10 mode=aggressive precision=f32
"""

# Runnable specs with finite, non-zero results: the CLI cannot fill data, so
# the specs above leave m zero (their wavefields are inf/NaN); these use
# constant coefficients and a constant forcing term instead.
ACOUSTIC_3D_FORCED = """\
grid shape=(20, 18, 22) extent=(190.0, 170.0, 210.0)
function damp space_order=8
timefunction u space_order=8 time_order=2
sparsetimefunction rec npoint=3 coords=((20.0, 30.0, 15.0), (100.5, 60.25, 33.0), (180.0, 160.0, 200.0))
eq u.forward = solve(0.25*u.dt2 - u.laplace + damp*u.dt - 1.5, u.forward)
rec.interpolate(u)
params steps=6 mode=advanced precision=f32
"""

ACOUSTIC_1D_FORCED = """\
grid shape=(21,) extent=(20.0,)
timefunction u space_order=4 time_order=2
sparsetimefunction rec npoint=2 coords=((3.3,), (12.75,))
eq u.forward = solve(2*u.dt2 - u.laplace - 0.5, u.forward)
rec.interpolate(u)
params steps=8 mode=basic precision=f64
"""

SNAPSHOT_2D_FORCED = """\
grid shape=(16, 15)
timefunction u space_order=4 time_order=2
timefunction us space_order=4 save=4 factor=3
eq u.forward = solve(u.dt2 - u.laplace - 0.25, u.forward)
eq us = u
params steps=10 mode=aggressive precision=f32
"""

EXPRESSIONS = [
    "grid shape=(11,)\ntimefunction u\neq u.forward = u + 0.5*u.dx\n",
    "grid shape=(11,) extent=(10.0,) origin=(1.0,)\nfunction f\n"
    "eq f = sin(f) + sqrt(f + 2)\n",
    "grid shape=(9, 9)\ntimefunction u\n"
    "eq u.forward = u.dx2 + u.dy2 region=interior\n",
    "grid shape=(9, 9)\nfunction a\nfunction b\n"
    "eq a = -b**2 - (a - b)/3 * cos(-b) + h_x*o_y - 2**-1\n",
    "grid shape=(8, 8, 8)\ntimefunction u space_order=4\n"
    "eq u.forward = 2*u - u.backward + dt**2*(u.dx2 + u.dy2 + u.dz2)\n",
]


def corpus():
    specs = [ACOUSTIC_1D, ACOUSTIC_3D, SNAPSHOT_2D] + EXPRESSIONS
    for shape, coords in (("(21,)", "((5.0,),)"), ("(12, 14)", "((5.0, 5.0),)")):
        for so in (2, 4):
            for mode in ("basic", "advanced", "aggressive"):
                specs.append(
                    "grid shape=%s\nfunction m space_order=%d\n"
                    "timefunction u space_order=%d time_order=2\n"
                    "sparsetimefunction src npoint=1 coords=%s\n"
                    "eq u.forward = solve(m*u.dt2 - u.laplace, u.forward)\n"
                    "src.inject(field=u.forward, expr=src * dt**2 / m)\n"
                    "params steps=5 mode=%s\n" % (shape, so, so, coords, mode))
    return specs


# (spec text, expected message fragment, line)
ERRORS = [
    ("grid shape=(11,)\ntimefunction u\neq u = u.dq\n", "unknown dimension q", 3),
    ("grid shape=(11,)\ntimefunction u\neq u = v + 1\n",
     "undeclared identifier 'v'", 3),
    ("grid shape=(11,)\ntimefunction u\neq u = (u +\n", "expected", 3),
    ("function m\n", "no grid declared", 1),
    ("grid shape=(11,)\nfunction m\nfunction m\n", "duplicate name 'm'", 3),
    ("grid shape=(11,)\ntimefunction u\neq u = u**0.5\n",
     "exponent must be an integer", 3),
    ("grid shape=(11,)\nfunction m\nparams speed=3\n",
     "unknown parameter 'speed'", 3),
    ("grid shape=(11,)\nfunction m\nbogus m\n", "unknown statement 'bogus'", 3),
    ("grid shape=(11,)\ntimefunction u\neq u.dx = u\n",
     "only .forward/.backward allowed on the left", 3),
    ("grid shape=(11,)\ntimefunction u\neq u = tan(u)\n", "unknown call 'tan'", 3),
]
