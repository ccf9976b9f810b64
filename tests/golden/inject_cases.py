"""Colliding-source injection case: 4096 sources on a
48^3 grid, half of them drawn from 256 shared positions (exact duplicates
and shared corners), half uniform. ``build(S, nsrc)`` takes a symbolic
module (the reference's or ours); ``fill`` writes the seeded inputs."""

import numpy as np

N, H_SP, SO = 48, 10.0, 4


def geometry(nsrc=4096, seed=5):
    rng = np.random.default_rng(seed)
    ext = H_SP * (N - 1)
    base = rng.uniform(0.3 * ext, 0.7 * ext, (256, 3))
    pts = np.concatenate([base[rng.integers(0, 256, nsrc // 2)],
                          rng.uniform(0.1 * ext, 0.9 * ext,
                                      (nsrc - nsrc // 2, 3))])
    src = [tuple(map(float, p)) for p in pts]
    rec = [(ext / 2, ext / 3, 40.0), (ext / 4, ext / 2, 100.0)]
    return src, rec


def build(S, nsrc=4096):
    import workloads
    src, rec = geometry(nsrc)
    return workloads.acoustic_equations((N, N, N), H_SP, SO, src, rec, S=S)


def fill(bufs, seed=6):
    import workloads
    rng = np.random.default_rng(seed)
    bufs["m"].data[...] = np.float32(1 / 2.0 ** 2)
    bufs["damp"].data[...] = workloads.damping_profile(
        (N, N, N), 4, SO // 2).astype(np.float32)
    bufs["src"].data[...] = rng.uniform(-1, 1, bufs["src"].data.shape)


DT = 0.4 * H_SP / 2.0
