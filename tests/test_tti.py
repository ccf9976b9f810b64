"""TTI: the operator authored with the reference API
(operators.tti_equations) is recognised for the fused kernel; the oracle
port reproduces the REAL reference bit for bit on it (goldens from
tests/golden/make_golden_tti.py); the GPU path agrees with the reference
within the north-star tolerance (rel-L2 <= 1e-5 wavefields, <= 1e-4 traces)."""

import hashlib
import json
import os

import numpy as np
import pytest

import tti_cases
import oracle
import paper_1807_03032_b200.symbolic as S
from paper_1807_03032_b200.backend.operator import Operator

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden():
    with open(os.path.join(GOLD, "tti.json")) as f:
        return json.load(f)


def _arrays(name):
    return np.load(os.path.join(GOLD, "arrays", name + ".npz"))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_tti_recognised_and_dse_bypassed():
    case = tti_cases.case_dict(tti_cases.CASES[0])
    op = Operator(tti_cases.build(S, case), dtype="f32")
    fused = [c for c in op.clusters if c.fused is not None]
    assert len(fused) == 1 and fused[0].fused[0] == "tti"
    roles = fused[0].fused[1]
    assert roles["theta"].name == "theta" and roles["m"].name == "m"


def test_tti_oracle_port_matches_reference_so4():
    case = tti_cases.case_dict(tti_cases.CASES[0])
    op = Operator(tti_cases.build(S, case), mode="advanced", dtype="f32",
                  fuse=False)
    trees = [repr((e.lhs, e.rhs)) for c in op.clusters for e in c.eqs]
    ref = _golden()["cases"][case["name"]]
    assert hashlib.sha256("\n".join(trees).encode()).hexdigest() == \
        ref["trees_sha"]
    bufs = op.allocate(case["nt"], pinned=False)
    tti_cases.fill(bufs, case)
    out = oracle.apply(op, case["nt"], bufs, dt=tti_cases.dt_of(case))
    for k in ("p", "r", "rec"):
        assert _sha(out[k]) == ref[k]["sha"], k


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.gpu
@pytest.mark.parametrize("row", tti_cases.CASES, ids=[c[0] for c in tti_cases.CASES])
def test_tti_gpu_vs_reference(row):
    case = tti_cases.case_dict(row)
    op = Operator(tti_cases.build(S, case), dtype="f32")
    bufs = op.allocate(case["nt"])
    tti_cases.fill(bufs, case)
    _, rep = op.apply(steps=case["nt"], buffers=bufs, dt=tti_cases.dt_of(case))
    assert [v for v in rep.values() if "fast_path" in v][0]["fast_path"]
    ref = _arrays(case["name"])
    for k in ("p", "r"):
        e32, e64 = _rel(bufs[k].data, ref[k]), _rel(bufs[k].data, ref[k + "64"])
        floor = _rel(ref[k], ref[k + "64"])
        assert e32 <= 1e-5 and e64 <= 1e-5, (k, e32, e64, floor)
    rec, r32 = bufs["rec"].data, ref["rec"]
    den = max(np.linalg.norm(r32), 1e-3 * np.abs(ref["rec64"]).max() *
              np.sqrt(r32.size))
    assert np.linalg.norm(rec - r32) / den <= 1e-4


with open(os.path.join(GOLD, "tti_long.json")) as _f:
    LONG_GOLD = json.load(_f)["cases"]


@pytest.mark.gpu
@pytest.mark.parametrize("row", tti_cases.LONG, ids=[c[0] for c in tti_cases.LONG])
def test_tti_gpu_vs_reference_long_horizon(row):
    """Every TTI order (so 4/8/12/16, 40^3, 100 steps) and config 3's
    horizon (so 8/12, 24^3, 500 steps) against the REAL reference run in f32
    and f64 (tests/golden/make_golden_tti_long.py). The reference's own f32
    result is itself ~1e-5 (100 steps) to ~1e-4 (500 steps) away from its f64
    result (``floor``), so the bar is relative to that floor: the GPU result
    must be as close to the f64 reference as the reference's own f32 run
    (within 1.5x its floor), and within 2x the floor of the f32 reference
    (two independently rounded f32 runs). Traces: <= 1e-4 (floored
    denominator, as above). The numbers are printed (pytest -s) and reported
    in DESIGN.md."""
    case = tti_cases.case_dict(row)
    gold = LONG_GOLD[case["name"]]
    ref = _arrays(case["name"])
    op = Operator(tti_cases.build(S, case), dtype="f32")
    bufs = op.allocate(case["nt"])
    tti_cases.fill(bufs, case)
    _, rep = op.apply(steps=case["nt"], buffers=bufs, dt=tti_cases.dt_of(case))
    assert [v for v in rep.values() if "fast_path" in v][0]["fast_path"]
    N, H = case["N"], case["so"] // 2
    inner = (gold["final_slot"],) + (slice(H, H + N),) * 3
    lines = []
    for k in ("p", "r"):
        got = bufs[k].data[inner]
        e32, e64 = _rel(got, ref[k]), _rel(got, ref[k + "64"])
        floor = gold[k]["floor_f32_vs_f64"]
        lines.append("%s %s: vs f32 %.3g, vs f64 %.3g, reference floor %.3g"
                     % (case["name"], k, e32, e64, floor))
        assert e64 <= 1.5 * floor + 1e-7, lines[-1]
        assert e32 <= 2.0 * floor + 1e-7, lines[-1]
    rec, r32, r64 = bufs["rec"].data, ref["rec"], ref["rec64"]
    den = max(np.linalg.norm(r32), 1e-3 * np.abs(r64).max() * np.sqrt(r32.size))
    erec = np.linalg.norm(rec - r32) / den
    lines.append("%s rec: vs f32 %.3g (floored)" % (case["name"], erec))
    print("\n".join(lines))
    assert erec <= 1e-4, lines[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("row", tti_cases.LONG[:4], ids=[c[0] for c in tti_cases.LONG[:4]])
def test_tti_gpu_f64_vs_reference_f64(row):
    """The f64 TTI path (same discretisation, double arithmetic) against the
    reference's own f64 run after 100 steps: agreement to ~1e-12 shows the
    kernels implement exactly the reference's equations (the f32 gaps above
    are rounding, not modelling)."""
    case = dict(tti_cases.case_dict(row), dtype="f64")
    gold = LONG_GOLD[case["name"]]
    ref = _arrays(case["name"])
    op = Operator(tti_cases.build(S, case), dtype="f64")
    bufs = op.allocate(case["nt"])
    tti_cases.fill(bufs, case)
    _, rep = op.apply(steps=case["nt"], buffers=bufs, dt=tti_cases.dt_of(case))
    assert [v for v in rep.values() if "fast_path" in v][0]["fast_path"]
    N, H = case["N"], case["so"] // 2
    inner = (gold["final_slot"],) + (slice(H, H + N),) * 3
    for k in ("p", "r"):
        e = _rel(bufs[k].data[inner], ref[k + "64"])
        print("%s f64 %s: vs ref f64 %.3g" % (case["name"], k, e))
        assert e <= 1e-10, (k, e)
    e = _rel(bufs["rec"].data, ref["rec64"])
    assert e <= 1e-10, ("rec", e)


def _build_nosparse(case):
    """The TTI p/r system alone (no source or receivers) on the case grid."""
    N, so = case["N"], case["so"]
    ext = tti_cases.H_SPACING * (N - 1)
    g = S.Grid((N,) * 3, extent=(ext,) * 3)
    p = S.FunctionDecl("p", "timefunction", g, space_order=so)
    r = S.FunctionDecl("r", "timefunction", g, space_order=so)
    f = {n: S.FunctionDecl(n, "function", g, space_order=so)
         for n in ("m", "damp", "epsilon", "delta", "theta", "phi")}
    return tti_cases.OPS.tti_equations(p, r, f["m"], f["damp"], f["epsilon"],
                                       f["delta"], f["theta"], f["phi"], S=S)


def _fill_nosparse(bufs, case):
    # tti_cases.fill also writes the source trace; give it a stub
    class _Stub:
        data = np.zeros((case["nt"], 1))
    tti_cases.fill(dict(bufs, src=_Stub()), case)


def test_tti_numpy_restatement_matches_oracle_so4():
    """Pins tests/tti_numpy.py (the high-order checker) to the oracle port
    (itself pinned bit for bit to the reference) on a so=4 f64 case."""
    import tti_numpy
    case = dict(name="np4", N=12, so=4, dtype="f64", nt=3, nrec=0)
    op = Operator(_build_nosparse(case), mode="advanced", dtype="f64",
                  fuse=False)
    bufs = op.allocate(case["nt"], pinned=False)
    _fill_nosparse(bufs, case)
    h = (tti_cases.H_SPACING,) * 3
    P, Rr = tti_numpy.run(bufs, 4, h, tti_cases.dt_of(case), case["nt"])
    out = oracle.apply(op, case["nt"], bufs, dt=tti_cases.dt_of(case))
    assert _rel(P, out["p"]) < 1e-12 and _rel(Rr, out["r"]) < 1e-12


# so 12/16 and odd extents (x-blocked TMA kernels with a ragged last pair,
# partial y/z tiles): GPU vs the float64 restatement (tests/tti_numpy.py)
EXTRA = [("tti_so12_f32_n21", 21, 12, "f32", 4),
         ("tti_so16_f32_n18", 18, 16, "f32", 3),
         ("tti_so12_f32_n40", 40, 12, "f32", 3),
         ("tti_so12_f64_n17", 17, 12, "f64", 3),
         # even storage extents: the z-pair pass-2 kernel (partial tiles)
         ("tti_so8_f32_n34", 34, 8, "f32", 3),
         ("tti_so4_f32_n46", 46, 4, "f32", 4)]


@pytest.mark.gpu
@pytest.mark.parametrize("row", EXTRA, ids=[c[0] for c in EXTRA])
def test_tti_gpu_high_order(row):
    import tti_numpy
    case = dict(zip(("name", "N", "so", "dtype", "nt"), row), nrec=0)
    op = Operator(_build_nosparse(case), dtype=case["dtype"])
    bufs = op.allocate(case["nt"])
    _fill_nosparse(bufs, case)
    h = (tti_cases.H_SPACING,) * 3
    P, Rr = tti_numpy.run(bufs, case["so"], h, tti_cases.dt_of(case),
                          case["nt"])
    _, rep = op.apply(steps=case["nt"], buffers=bufs, dt=tti_cases.dt_of(case))
    assert [v for v in rep.values() if "fast_path" in v][0]["fast_path"]
    tol = 1e-5 if case["dtype"] == "f32" else 1e-12
    for k, ref in (("p", P), ("r", Rr)):
        e = _rel(bufs[k].data, ref)
        assert e <= tol, (k, e)


# the opt-in coupled single launch (SC_TTI_COUPLED=1: both passes, g through
# L2) against the two launches: same arithmetic, so bit for bit; one to three
# rounds of tiles, partial tiles, every order it serves
COUPLED = [("so12_n40", 40, 12, 5), ("so12_n75", 75, 12, 4),
           ("so8_n70", 70, 8, 4), ("so4_n90", 90, 4, 4),
           ("so12_n300", 300, 12, 3), ("so8_n250", 250, 8, 2)]


@pytest.mark.gpu
@pytest.mark.parametrize("row", COUPLED, ids=[c[0] for c in COUPLED])
def test_tti_coupled_launch_equals_two_launches(row, monkeypatch):
    case = dict(zip(("name", "N", "so", "nt"), row), dtype="f32", nrec=0)
    outs = []
    for two in (False, True):
        if two:
            monkeypatch.delenv("SC_TTI_COUPLED", raising=False)
        else:
            monkeypatch.setenv("SC_TTI_COUPLED", "1")
        op = Operator(_build_nosparse(case), dtype="f32")
        bufs = op.allocate(case["nt"])
        _fill_nosparse(bufs, case)
        _, rep = op.apply(steps=case["nt"], buffers=bufs,
                          dt=tti_cases.dt_of(case))
        assert [v for v in rep.values() if "fast_path" in v][0]["fast_path"]
        outs.append({k: bufs[k].data.copy() for k in ("p", "r")})
    for k in ("p", "r"):
        assert np.isfinite(outs[0][k]).all() and np.abs(outs[0][k]).max() > 0
        assert np.array_equal(outs[0][k], outs[1][k]), k


@pytest.mark.gpu
def test_tti_config3_full_size_linearity():
    """BASELINE config 3 at its full grid (592^3, so=12): the step is linear
    in the wavefields and the source, and scaling by 2 is exact in floating
    point, so doubling the initial p, r and the source trace must double
    the result bit for bit (a size-independent check of the fused passes,
    their TMA rings and chunking at full size; values within tolerance of
    the reference are checked on the reduced grids above)."""
    import workloads
    op, bufs, dt, meta = workloads.config3(so=12, nt=8)
    rng = np.random.default_rng(12)
    H = 6
    for k in ("p", "r"):
        inner = bufs[k].data[0:2, H:-H, H:-H, H:-H]
        inner[...] = rng.uniform(-1, 1, inner.shape).astype(np.float32)
    twice = {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
             for k, b in bufs.items()}
    for k in ("p", "r", "src"):
        twice[k].data[...] *= 2
    _, rep = op.apply(steps=meta["nt"], buffers=bufs, dt=dt)
    assert [v for v in rep.values() if "fast_path" in v][0]["fast_path"]
    op.apply(steps=meta["nt"], buffers=twice, dt=dt)
    for k in ("p", "r"):
        a, b = bufs[k].data, twice[k].data
        assert np.isfinite(a).all() and np.abs(a).max() > 0
        assert np.array_equal(2 * a, b), k
