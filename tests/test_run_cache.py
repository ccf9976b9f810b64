"""Prepared-run reuse across applies (Operator.apply keeps one prepared run:
device buffers, programs, CUDA graph). Reuse must be invisible: results equal
fresh prepares bit for bit, and any change to a host value that fed a
per-point table, or to data that breaks a fused kernel's precondition,
forces a fresh prepare."""

import numpy as np
import pytest

import oracle
import workloads
from paper_1807_03032_b200.backend import operator as opmod

pytestmark = pytest.mark.gpu


def _copy(bufs):
    return {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
            for k, b in bufs.items()}


def _small(nt=6):
    return workloads.config2(so=8, n=40, nbl=6, nt=nt, nrec_side=12)


def _fresh(op, bufs, dt, nt, monkeypatch):
    monkeypatch.setenv("SC_NO_RUN_CACHE", "1")
    op.apply(nt, bufs, dt=dt)
    monkeypatch.delenv("SC_NO_RUN_CACHE")


def test_second_apply_reuses_and_matches(monkeypatch):
    op, bufs, dt, meta = _small()
    nt = meta["nt"]
    ref = _copy(bufs)
    op.apply(nt, bufs, dt=dt)
    run = opmod._RUN_CACHE["run"]
    assert run is not None and opmod._RUN_CACHE["op"] is op
    op.apply(nt, bufs, dt=dt)                    # continues from the result
    assert opmod._RUN_CACHE["run"] is run       # reused, not re-prepared
    _fresh(op, ref, dt, nt, monkeypatch)
    _fresh(op, ref, dt, nt, monkeypatch)
    for k in ("u", "rec"):
        assert np.array_equal(bufs[k].data, ref[k].data), k
    op.release()
    assert opmod._RUN_CACHE["run"] is None


def test_changed_coordinates_invalidate(monkeypatch):
    op, bufs, dt, meta = _small()
    nt = meta["nt"]
    op.apply(nt, bufs, dt=dt)
    run = opmod._RUN_CACHE["run"]
    bufs["rec_coords"].data[3] += 7.5           # new receiver position
    ref = _copy(bufs)
    op.apply(nt, bufs, dt=dt)
    assert opmod._RUN_CACHE["run"] is not run
    out = oracle.apply(op, nt, ref, dt=dt)
    assert np.array_equal(bufs["rec"].data, out["rec"])
    assert np.array_equal(bufs["u"].data, out["u"])


def test_precondition_rechecked_on_reuse():
    """m changed so the fused kernel's reciprocal precondition fails: the
    reused run must notice (sc_revalidate) and the exact generic program
    runs instead -- bitwise equal to the oracle."""
    op, bufs, dt, meta = _small()
    nt = meta["nt"]
    op.apply(nt, bufs, dt=dt)
    bufs["m"].data[20, 20, 20] = 1e-38          # interior, damp = 0
    ref = _copy(bufs)
    _, rep = op.apply(nt, bufs, dt=dt)
    sec = [v for v in rep.values() if "fast_path" in v][0]
    assert not sec["fast_path"]
    out = oracle.apply(op, nt, ref, dt=dt)
    a, b = bufs["u"].data, out["u"]
    assert np.array_equal(np.isnan(a), np.isnan(b))
    ok = ~np.isnan(a)
    assert np.array_equal(a[ok].view(np.uint32), b[ok].view(np.uint32))


def test_rec_not_uploaded_when_fully_overwritten():
    op, bufs, dt, meta = _small()
    nt = meta["nt"]
    op.apply(nt, bufs, dt=dt)
    run = opmod._RUN_CACHE["run"]
    assert "rec" in run.no_upload
    op.apply(nt, bufs, dt=dt, t_m=0, t_M=nt - 2)  # last row kept: uploaded
    run = opmod._RUN_CACHE["run"]
    assert "rec" not in run.no_upload
    op.release()


def test_dead_slot_uploads_only_its_halo_shell(monkeypatch):
    """u[t_m + 1] is overwritten over the whole loop box by the first step
    before anything reads it: a reused run uploads only that slot's halo
    shell (sc_upload_shell). Garbage in the dead interior must not matter,
    non-zero halo values must arrive, and the result equals the oracle and
    the full upload bit for bit."""
    op, bufs, dt, meta = _small()
    nt = meta["nt"]
    op.apply(nt, bufs, dt=dt)                     # prepares
    run = opmod._RUN_CACHE["run"]
    assert "u" in run.dead
    slot, lo, hi = run.dead["u"]
    assert slot == 1 and lo == [4, 4, 4]
    rng = np.random.default_rng(5)
    u = bufs["u"].data
    u[...] = rng.uniform(-1e-3, 1e-3, u.shape).astype(np.float32)   # halo shells too
    inner = u[slot, lo[0]:hi[0] + 1, lo[1]:hi[1] + 1, lo[2]:hi[2] + 1]
    inner[...] = np.float32(1e30)                 # dead on entry
    ref, full = _copy(bufs), _copy(bufs)
    op.apply(nt, bufs, dt=dt)
    assert opmod._RUN_CACHE["run"] is run
    box = np.prod([h - l + 1 for l, h in zip(lo, hi)])
    assert run.h2d_bytes < sum(b.data.nbytes for k, b in bufs.items()
                               if k in op.functions) - 4 * box + 4096
    out = oracle.apply(op, nt, ref, dt=dt)
    monkeypatch.setenv("SC_FULL_UPLOAD", "1")
    _fresh(op, full, dt, nt, monkeypatch)
    for k in ("u", "rec"):
        assert np.isfinite(bufs[k].data).all()
        assert np.array_equal(bufs[k].data, out[k]), k
        assert np.array_equal(bufs[k].data, full[k].data), k
    op.release()


def test_early_download_of_final_receiver_rows(monkeypatch):
    """Receiver rows are final once their step is done: apply starts their
    device->host copy before the loop ends (sc_early_download) and
    download() copies the rest. Same bits as without it and as the oracle,
    on the first (preparing) apply and on a reused run."""
    op, bufs, dt, meta = workloads.config2(so=8, n=40, nbl=6, nt=96,
                                           nrec_side=12)
    nt = meta["nt"]
    ref, plain = _copy(bufs), _copy(bufs)
    op.apply(nt, bufs, dt=dt)
    run = opmod._RUN_CACHE["run"]
    first = {k: bufs[k].data.copy() for k in ("u", "rec")}
    again = op.allocate(nt)                       # page-locked, like bufs
    for k, b in again.items():
        b.data[...] = ref[k].data
    early = []
    orig = type(run).download

    def spy(self, *a, **k):
        early.append(getattr(self, "_early", None))
        return orig(self, *a, **k)
    monkeypatch.setattr(type(run), "download", spy)
    op.apply(nt, again, dt=dt)                    # reused run
    assert opmod._RUN_CACHE["run"] is run
    assert early and early[-1] is not None and early[-1][0] == "rec"
    assert 0 < early[-1][1] < nt
    monkeypatch.setenv("SC_NO_EARLY_D2H", "1")
    _fresh(op, plain, dt, nt, monkeypatch)
    out = oracle.apply(op, nt, ref, dt=dt)
    for k in ("u", "rec"):
        assert np.array_equal(first[k], out[k]), k
        assert np.array_equal(again[k].data, out[k]), k
        assert np.array_equal(plain[k].data, out[k]), k
    op.release()


def test_tti_reused_run_matches_fresh_prepares(monkeypatch):
    """The fused TTI path through a reused run: p and r each have a slot
    that is dead on entry (halo-shell upload), and the traces leave early.
    Two applies in a row (the second continues from the first) equal two
    fresh prepares bit for bit."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import tti_cases
    import paper_1807_03032_b200.symbolic as S
    from paper_1807_03032_b200.backend.operator import Operator
    case = dict(tti_cases.case_dict(tti_cases.LONG[2]), nt=70)   # so 12, 40^3
    op = Operator(tti_cases.build(S, case), dtype="f32")
    nt, dt = case["nt"], tti_cases.dt_of(case)
    bufs = op.allocate(nt)
    tti_cases.fill(bufs, case)
    rng = np.random.default_rng(3)
    for k in ("p", "r"):                          # non-zero halo shells
        bufs[k].data[...] += rng.uniform(-1e-6, 1e-6, bufs[k].data.shape
                                         ).astype(np.float32)
    ref = _copy(bufs)
    op.apply(nt, bufs, dt=dt)
    run = opmod._RUN_CACHE["run"]
    assert set(run.dead) == {"p", "r"}
    op.apply(nt, bufs, dt=dt)
    assert opmod._RUN_CACHE["run"] is run
    _fresh(op, ref, dt, nt, monkeypatch)
    _fresh(op, ref, dt, nt, monkeypatch)
    for k in ("p", "r", "rec"):
        assert np.isfinite(bufs[k].data).all()
        assert np.array_equal(bufs[k].data, ref[k].data), k
    op.release()


def test_early_download_on_the_graph_path():
    """run(profile=False) launches the captured graph; with the early trace
    download the loop is two graphs with the copy started between them
    (sc_early_download). Same bits as the oracle, twice in a row."""
    op, bufs, dt, meta = workloads.config2(so=8, n=40, nbl=6, nt=96,
                                           nrec_side=12)
    nt = meta["nt"]
    ref = _copy(bufs)
    run = op.prepare(nt, bufs, dt=dt)
    try:
        run.run(profile=False, early_download=True)
        assert run._early is not None and run._early[0] == "rec"
        run.download()
        out = oracle.apply(op, nt, ref, dt=dt)
        for k in ("u", "rec"):
            assert np.array_equal(bufs[k].data, out[k]), k
        run.rebind(bufs)                          # continue from the result
        run.run(profile=False, early_download=True)
        run.download()
        ref2 = {k: type(b)(b.name, b.dtype, b.extents, data=out[k].copy()
                           if k in out else b.data.copy())
                for k, b in ref.items()}
        out2 = oracle.apply(op, nt, ref2, dt=dt)
        for k in ("u", "rec"):
            assert np.array_equal(bufs[k].data, out2[k]), k
        run.run(profile=False)                    # disarmed again
        assert run._early is None
    finally:
        run.close()
