"""Run one golden case on the GPU and report bitwise parity (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import numpy as np
import cases, oracle
from helpers import CASES, golden, make, sha

name = sys.argv[1]
fast = os.environ.get("SC_NOFAST")
c = CASES[name]
op, bufs = make(c)
_, rep = op.apply(steps=c["nt"], buffers=bufs, dt=cases.dt_of(c))
ref = golden()["cases"][name]
ok = all(sha(bufs[k].data) == v["sha"] for k, v in ref.items()
         if k in ("u", "rec") or k.startswith("temp"))
sec = [s for s in rep.values() if "launches" in s][0]
print(name, "OK" if ok else "MISMATCH", "fast", sec["fast_path"], "%.3f ms" % (sec["time"] * 1e3))
