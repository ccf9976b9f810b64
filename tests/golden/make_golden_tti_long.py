"""Long-horizon TTI fixtures from the REAL reference (build container only).

Every TTI order (so 4/8/12/16) at 40^3 over 100 steps, plus so 8/12 at
24^3 over config 3's nt = 500, each in f32 AND f64 (tests/golden/
tti_cases.LONG, "stable" fill: delta = min(delta, epsilon)). The reference's
advanced-mode DSE takes 10 s (so 4) to ~16 min (so 16) per compile
(SURVEY.md §0.1 #2), so every (case, dtype) runs in its own process:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_tti_long.py run NAME DTYPE
    python tests/golden/make_golden_tti_long.py merge

``run`` writes tests/golden/tti_long/NAME_DTYPE.npz (scratch, git-ignored);
``merge`` writes tests/golden/tti_long.json (digests, norms, the f32-vs-f64
floor of the reference itself) and arrays/NAME.npz with the final time level
of p and r (interior, f32 run and f64 run) and the full traces of both runs.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
SCRATCH = os.path.join(HERE, "tti_long")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(name, dtype):
    REF = os.environ.get("REF", "/root/reference")
    sys.path.insert(0, os.path.join(REF, "pkg", "src"))
    import tti_cases
    import stencilc.symbolic as S
    from stencilc.backend.operator import Operator
    row = [r for r in tti_cases.LONG if r[0] == name][0]
    case = dict(tti_cases.case_dict(row), dtype=dtype)
    t0 = time.time()
    op = Operator(tti_cases.build(S, case), mode="advanced", dtype=dtype)
    tc = time.time() - t0
    bufs = op.allocate(case["nt"])
    tti_cases.fill(bufs, case)
    t0 = time.time()
    op.apply(steps=case["nt"], buffers=bufs, dt=tti_cases.dt_of(case))
    ta = time.time() - t0
    trees = [repr((e.lhs, e.rhs)) for c in op.artifact.clusters for e in c.eqs]
    os.makedirs(SCRATCH, exist_ok=True)
    np.savez(os.path.join(SCRATCH, "%s_%s.npz" % (name, dtype)),
             p=bufs["p"].data, r=bufs["r"].data, rec=bufs["rec"].data,
             meta=np.array(json.dumps({
                 "compile_s": tc, "apply_s": ta, "numpy": np.__version__,
                 "trees_sha": hashlib.sha256("\n".join(trees).encode())
                 .hexdigest()})))
    print(name, dtype, "compile %.1fs apply %.1fs" % (tc, ta), flush=True)


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def merge():
    import tti_cases
    out = {"numpy": np.__version__, "note": __doc__.split("\n")[0],
           "cases": {}}
    for row in tti_cases.LONG:
        name, N, so, _, nt, _ = row
        d32 = np.load(os.path.join(SCRATCH, name + "_f32.npz"))
        d64 = np.load(os.path.join(SCRATCH, name + "_f64.npz"))
        H = so // 2
        last = nt % 3
        inner = (last, slice(H, H + N), slice(H, H + N), slice(H, H + N))
        m32 = json.loads(str(d32["meta"]))
        m64 = json.loads(str(d64["meta"]))
        entry = {"final_slot": last, "compile_s": [m32["compile_s"],
                                                   m64["compile_s"]],
                 "apply_s": [m32["apply_s"], m64["apply_s"]],
                 "trees_sha": m32["trees_sha"]}
        arrays = {}
        for k in ("p", "r"):
            a32, a64 = d32[k][inner], d64[k][inner]
            entry[k] = {"sha_full_f32": sha(d32[k]), "l2": float(
                np.linalg.norm(a32.astype(np.float64))),
                "l2_f64": float(np.linalg.norm(a64)),
                "floor_f32_vs_f64": _rel(a32, a64)}
            arrays[k] = a32
            arrays[k + "64"] = a64
        arrays["rec"] = d32["rec"]
        arrays["rec64"] = d64["rec"]
        entry["rec"] = {"sha_f32": sha(d32["rec"]),
                        "floor_f32_vs_f64": _rel(d32["rec"], d64["rec"])}
        np.savez_compressed(os.path.join(HERE, "arrays", name + ".npz"),
                            **arrays)
        out["cases"][name] = entry
        print(name, entry["p"]["floor_f32_vs_f64"],
              entry["r"]["floor_f32_vs_f64"], entry["rec"]["floor_f32_vs_f64"])
    with open(os.path.join(HERE, "tti_long.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        merge()
