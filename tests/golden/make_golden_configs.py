"""Config-size acoustic digests from the REAL reference (build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_configs.py [name ...]

BASELINE config 1 at its full size (148^3, so=4, nt=200, 101 receivers; the
centre source and the shallow parity variant of SURVEY.md §8d) and config 2's
full 592^3 grid (so 8/12/16) over a few steps with a 32 x 32 receiver subset
and a random initial wavefield. Inputs come from workloads.py (the same
generator the GPU tests use), are copied into the reference's own buffers,
and the reference's Operator.apply runs with all host threads (its results
are bitwise independent of ``workers``, reference test_backend.py:166-171).
Writes tests/golden/configs.json: sha256 of the final u and rec.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF = os.environ.get("REF", "/root/reference")
sys.path.insert(0, os.path.join(REF, "pkg", "src"))

import workloads  # noqa: E402
import stencilc.symbolic as RS  # noqa: E402
from stencilc.backend.operator import Operator as RefOp  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def config1(src_depth):
    return workloads.config1(src_depth=src_depth)


def config2(so):
    op, bufs, dt, meta = workloads.config2(so=so, nt=3, nrec_side=32)
    workloads.seed_interior(bufs, so, seed=3)
    return op, bufs, dt, meta


CASES = {
    "config1_centre": lambda: config1(None),
    "config1_shallow": lambda: config1(320.0),
    "config2_so8_nt3": lambda: config2(8),
    "config2_so12_nt3": lambda: config2(12),
    "config2_so16_nt3": lambda: config2(16),
}


def run(name):
    op, bufs, dt, meta = CASES[name]()
    eqs = workloads.acoustic_equations(meta["shape"], meta["h"], meta["so"],
                                       meta["src_coords"], meta["rec_coords"],
                                       S=RS)
    ref = RefOp(eqs, mode="advanced", dtype="f32")
    rb = ref.allocate(meta["nt"])
    for k, b in bufs.items():
        if k in rb and not k.endswith("_coords"):
            rb[k].data[...] = b.data
    for k in ("src_coords", "rec_coords"):
        assert np.array_equal(rb[k].data, bufs[k].data), k
    t0 = time.time()
    ref.apply(steps=meta["nt"], buffers=rb, dt=dt, workers=os.cpu_count())
    el = time.time() - t0
    out = {"u": sha(rb["u"].data), "rec": sha(rb["rec"].data),
           "u_l2": float(np.linalg.norm(rb["u"].data.astype(np.float64))),
           "rec_maxabs": float(np.abs(rb["rec"].data).max()),
           "shape": list(meta["shape"]), "so": meta["so"], "nt": meta["nt"],
           "nrec": meta["nrec"], "apply_s": el}
    print(name, out, flush=True)
    return out


def main():
    names = sys.argv[1:] or list(CASES)
    path = os.path.join(HERE, "configs.json")
    db = {"numpy": np.__version__, "cases": {}}
    if os.path.exists(path):
        with open(path) as f:
            db = json.load(f)
    for n in names:
        db["cases"][n] = run(n)
        with open(path, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
