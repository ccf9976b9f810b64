"""Source injection (reference sparse.py:52-71 and the
ATOMIC point loop iet.py:234-245). Targets that collide (sources sharing
corners) are applied by a target-grouped kernel: one thread per distinct
target folds its increments in the oracle's (point, corner) order, so the
result is bitwise the serial loop's while running in parallel.
SC_INJECT_ATOMIC=1 selects hardware atomics (tolerance mode)."""

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


def _colliding(nsrc=4096, n=48, nt=8, seed=5):
    rng = np.random.default_rng(seed)
    h = 10.0
    N = n
    ext = h * (N - 1)
    # half the sources on 256 shared positions (many exact duplicates and
    # shared corners), half uniformly random
    base = rng.uniform(0.3 * ext, 0.7 * ext, (256, 3))
    pts = np.concatenate([base[rng.integers(0, 256, nsrc // 2)],
                          rng.uniform(0.1 * ext, 0.9 * ext, (nsrc - nsrc // 2, 3))])
    src = [tuple(map(float, p)) for p in pts]
    rec = [(ext / 2, ext / 3, 40.0), (ext / 4, ext / 2, 100.0)]
    op = workloads.acoustic_operator((N, N, N), h, 4, src, rec)
    bufs = op.allocate(nt)
    bufs["m"].data[...] = np.float32(1 / 2.0 ** 2)
    bufs["damp"].data[...] = workloads.damping_profile(
        (N, N, N), 4, 2).astype(np.float32)
    dt = 0.4 * h / 2.0
    bufs["src"].data[...] = rng.uniform(-1, 1, bufs["src"].data.shape)
    return op, bufs, dt, nt


def _copy(bufs):
    return {k: type(b)(b.name, b.dtype, b.extents, data=b.data.copy())
            for k, b in bufs.items()}


def test_colliding_injection_bitwise_and_fast():
    op, bufs, dt, nt = _colliding()
    ref = _copy(bufs)
    _, rep = op.apply(nt, bufs, dt=dt)
    sec = [v for v in rep.values() if "stages" in v][0]
    inj = [v for k, v in sec["stages"].items() if k.startswith("sparse")][0]
    out = oracle.apply(op, nt, ref, dt=dt)
    assert np.array_equal(bufs["u"].data, out["u"])
    assert np.array_equal(bufs["rec"].data, out["rec"])
    per_step_us = inj / nt * 1e6
    print("colliding injection, 4096 sources: %.1f us/step" % per_step_us)
    assert per_step_us < 50.0
    op.release()


def test_colliding_injection_atomic_tolerance(monkeypatch):
    monkeypatch.setenv("SC_INJECT_ATOMIC", "1")
    op, bufs, dt, nt = _colliding(nsrc=1024)
    ref = _copy(bufs)
    op.apply(nt, bufs, dt=dt)
    out = oracle.apply(op, nt, ref, dt=dt)
    a = bufs["u"].data.astype(np.float64)
    b = out["u"].astype(np.float64)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5
    op.release()
