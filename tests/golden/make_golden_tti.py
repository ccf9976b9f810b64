"""TTI golden fixtures from the REAL reference (build container only; the
advanced-mode compile of so=8 takes ~80 s in the reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_tti.py
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
REF = os.environ.get("REF", "/root/reference")
sys.path.insert(0, os.path.join(REF, "pkg", "src"))

import tti_cases  # noqa: E402
import stencilc.symbolic as S  # noqa: E402
from stencilc.backend.operator import Operator  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"numpy": np.__version__, "cases": {}}
    for row in tti_cases.CASES:
        case = tti_cases.case_dict(row)
        t0 = time.time()
        op = Operator(tti_cases.build(S, case), mode="advanced",
                      dtype=case["dtype"])
        tc = time.time() - t0
        bufs = op.allocate(case["nt"])
        tti_cases.fill(bufs, case)
        f64 = Operator(tti_cases.build(S, case), mode="advanced", dtype="f64")
        b64 = f64.allocate(case["nt"])
        tti_cases.fill(b64, dict(case, dtype="f64"))
        op.apply(steps=case["nt"], buffers=bufs, dt=tti_cases.dt_of(case))
        f64.apply(steps=case["nt"], buffers=b64, dt=tti_cases.dt_of(case))
        trees = [repr((e.lhs, e.rhs)) for c in op.artifact.clusters
                 for e in c.eqs]
        entry = {"compile_s": tc, "trees_sha": hashlib.sha256(
            "\n".join(trees).encode()).hexdigest()}
        for k in ("p", "r", "rec"):
            a = bufs[k].data
            entry[k] = {"sha": sha(a), "l2": float(np.linalg.norm(a)),
                        "l2_f64": float(np.linalg.norm(b64[k].data))}
        np.savez_compressed(os.path.join(HERE, "arrays", case["name"] + ".npz"),
                            p=bufs["p"].data, r=bufs["r"].data,
                            rec=bufs["rec"].data, p64=b64["p"].data,
                            r64=b64["r"].data, rec64=b64["rec"].data)
        out["cases"][case["name"]] = entry
        print(case["name"], "compile %.1fs" % tc, entry["p"]["l2"], flush=True)
    with open(os.path.join(HERE, "tti.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
