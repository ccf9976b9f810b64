"""Block-shape autotuner.

Restates the reference's tuner (reference ``backend/operator.py:256-272``
``autotune`` and ``iet.py:426-443`` ``autotune_blocks`` /
``default_block_candidates``): time each candidate block shape, return the
fastest, ties to the earliest candidate (deterministic for a fixed candidate
order).

On the B200 backend a block shape maps onto the launch geometry
(reference loop blocking, iet.py:377-423):

* ``x`` (3D) sets the x planes each CTA of the fused kernels streams (its x
  chunk: more planes amortise the re-read x halo, fewer give more CTAs per
  wave);
* the innermost and next space dimensions (``z`` and ``y`` in 3D, ``y``
  and ``x`` in 2D) set the thread-block extents of the NVRTC-generated
  kernels (csrc/jit.cu), which run every statement without a fused family
  kernel;
* the fused kernels' y/z tile is fixed by their register blocking.

Results never depend on the block shape (the same per-point arithmetic runs
in every chunking). Runs are timed on the device with CUDA events over
prepared runs (``DeviceRun.run`` reports the time loop).
"""

from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence

from .buffers import BackendError

BLOCK_SIZES = (4, 8, 16, 32, 64)


def autotune_blocks(iet, runner: Callable[[dict], float],
                    candidates: Sequence[dict]) -> dict:
    """The fastest candidate by ``runner`` (seconds); ties go to the earliest
    (reference iet.py:426-439). ``iet`` is accepted for signature parity."""
    if not candidates:
        raise BackendError("no block-shape candidates")
    best, best_time = None, None
    for cand in candidates:
        elapsed = runner(cand)
        if best_time is None or elapsed < best_time:
            best, best_time = cand, elapsed
    return best


def default_block_candidates(dims: Sequence[str]) -> List[dict]:
    """Same closed family as the reference (iet.py:442-443)."""
    return [{d: size for d in dims} for size in BLOCK_SIZES]


def device_runner(eqs, mode: str = "advanced", dtype: str = "f64",
                  steps: int = 3, buffers: Optional[Dict] = None,
                  repeats: int = 2, **params) -> Callable[[dict], float]:
    """A runner timing ``steps`` time steps of ``Operator(eqs, block=shape)``
    on the GPU: one prepared run per shape (compile, upload, graph capture
    excluded), launched ``repeats`` times, best device time (s)."""
    from .operator import Operator

    def run(shape: dict) -> float:
        op = Operator(eqs, mode=mode, block=shape, dtype=dtype)
        bufs = buffers if buffers is not None else op.allocate(steps)
        r = op.prepare(steps, bufs, **params)
        try:
            best = None
            for _ in range(max(1, repeats) + 1):   # first launch: capture
                rep = r.run(profile=False)
                sec = [v for v in rep.values() if "launches" in v]
                t = sum(v["time"] for v in sec)
                best = t if best is None else min(best, t)
            return best
        finally:
            r.close()

    return run


def autotune(eqs, mode: str = "advanced", dtype: str = "f64", steps: int = 3,
             candidates: Optional[Sequence[dict]] = None,
             buffers: Optional[Dict] = None, **params) -> dict:
    """Pick a block shape by timing short runs (reference operator.py:256-272:
    same signature; ``buffers`` and ``params`` (e.g. ``dt``) are passed to
    the timed runs, zeroed buffers by default)."""
    from .operator import Operator
    probe = Operator(eqs, mode=mode, dtype=dtype)
    dims = [d.name for d in probe.grid.dimensions]
    if candidates is None:
        candidates = default_block_candidates(dims)
    runner = device_runner(eqs, mode, dtype, steps, buffers, **params)
    return autotune_blocks(getattr(probe, "iet", None), runner,
                           list(candidates))
