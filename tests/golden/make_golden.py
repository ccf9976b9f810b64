"""Generate golden fixtures by running the REAL reference (pkg/src/stencilc)
in the build container. Not run on the GPU box (the reference is absent
there); its outputs are committed under tests/golden/.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes
* acoustic.json: per case, sha256 + stats of the final ``u`` and ``rec``
  buffers and of the hoisted sparse tables (temp*), plus the optimized
  trees' repr (to pin the restated lowering/DSE);
* arrays/<case>.npz: full final arrays for the smaller cases (diagnostics
  and tolerance tests).
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
REF = os.environ.get("REF", "/root/reference")
sys.path.insert(0, os.path.join(REF, "pkg", "src"))

import cases  # noqa: E402
import stencilc.symbolic as S  # noqa: E402
from stencilc.backend.operator import Operator  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"numpy": np.__version__, "python": sys.version.split()[0],
           "cases": {}}
    os.makedirs(os.path.join(HERE, "arrays"), exist_ok=True)
    for row in cases.CASES:
        case = cases.case_dict(row)
        eqs = cases.build(S, case)
        op = Operator(eqs, mode=case["mode"], dtype=case["dtype"])
        nt = case["nt"]
        bufs = op.allocate(nt)
        cases.fill(bufs, case)
        _, report = op.apply(steps=nt, buffers=bufs, dt=cases.dt_of(case))
        trees = [repr((e.lhs, e.rhs)) for c in op.artifact.clusters
                 for e in c.eqs]
        entry = {"trees_sha": hashlib.sha256("\n".join(trees).encode())
                 .hexdigest(), "sections": sorted(report)}
        for name in sorted(bufs):
            if name in ("u", "rec") or name.startswith("temp"):
                a = bufs[name].data
                entry[name] = {"sha": sha(a), "shape": list(a.shape),
                               "l2": float(np.linalg.norm(a.astype(np.float64))),
                               "max": float(np.abs(a).max())}
        np.savez_compressed(os.path.join(HERE, "arrays", case["name"] + ".npz"),
                            **{k: bufs[k].data for k in bufs
                               if k in ("u", "rec") or k.startswith("temp")})
        out["cases"][case["name"]] = entry
        print(case["name"], entry["u"]["l2"], entry["rec"]["l2"], flush=True)
    # Tree reprs for the acoustic family (lowering + DSE pinning)
    with open(os.path.join(HERE, "acoustic.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
