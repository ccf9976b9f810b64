"""Snapshot goldens from the REAL reference (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_snapshot.py
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

import snapshot_cases  # noqa: E402
import stencilc.symbolic as S  # noqa: E402
from stencilc.backend.operator import Operator  # noqa: E402


def main():
    out = {"numpy": np.__version__, "cases": {}}
    for row in snapshot_cases.CASES:
        case = snapshot_cases.case_dict(row)
        op = Operator(snapshot_cases.build(S, case), mode=case["mode"],
                      dtype=case["dtype"])
        bufs = op.allocate(case["steps"])
        snapshot_cases.fill(bufs, case)
        bufs, rep = op.apply(steps=case["steps"], buffers=bufs,
                             dt=snapshot_cases.DT)
        trees = [repr((e.lhs, e.rhs)) for c in op.artifact.clusters
                 for e in c.eqs]
        entry = {"trees_sha": hashlib.sha256("\n".join(trees).encode()).hexdigest(),
                 "points": {k: v["points"] for k, v in rep.items()}}
        arrs = {}
        for k in ("u", "us", "img"):
            a = bufs[k].data
            entry[k] = hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
            arrs[k] = a
        np.savez_compressed(os.path.join(HERE, "arrays", case["name"] + ".npz"),
                            **arrs)
        out["cases"][case["name"]] = entry
        print(case["name"], entry["points"], float(np.abs(arrs["img"]).max()))
    with open(os.path.join(HERE, "snapshot.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
