"""Colliding-injection digests from the REAL reference (build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_inject.py
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
REF = os.environ.get("REF", "/root/reference")
sys.path.insert(0, os.path.join(REF, "pkg", "src"))

import inject_cases  # noqa: E402
import stencilc.symbolic as S  # noqa: E402
from stencilc.backend.operator import Operator  # noqa: E402

NT = 8


def main():
    out = {"numpy": np.__version__, "cases": {}}
    for nsrc in (4096, 1024):
        op = Operator(inject_cases.build(S, nsrc), dtype="f32")
        bufs = op.allocate(NT)
        inject_cases.fill(bufs)
        op.apply(steps=NT, buffers=bufs, dt=inject_cases.DT)
        out["cases"]["collide_%d" % nsrc] = {
            k: hashlib.sha256(np.ascontiguousarray(bufs[k].data).tobytes())
            .hexdigest() for k in ("u", "rec")}
        print(nsrc, float(np.abs(bufs["u"].data).max()), flush=True)
    with open(os.path.join(HERE, "inject.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
