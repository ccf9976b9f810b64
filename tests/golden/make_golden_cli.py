"""CLI goldens from the REAL reference (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cli.py

For every corpus spec: the reference parser's signature() sha and equation
count; for the runnable specs, `stencilc run --dump` outputs (sha and the
arrays, small) and the printed section lines; for the error corpus the
reference's (message, line, col)."""

import hashlib
import io
import json
import os
import sys
import tempfile
from contextlib import redirect_stdout, redirect_stderr

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
REF = os.environ.get("REF", "/root/reference")
sys.path.insert(0, os.path.join(REF, "pkg", "src"))

import cli_corpus  # noqa: E402
from stencilc.cli.driver import main as ref_main  # noqa: E402
from stencilc.cli.parser import SpecError, parse_spec  # noqa: E402


def sig_sha(spec):
    return hashlib.sha256(repr(spec.signature()).encode()).hexdigest()


def run_dump(text, funcs, steps, dt):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "p.spec")
        with open(path, "w") as f:
            f.write(text)
        args = ["run", path, "--steps", str(steps), "--dt", repr(dt)]
        for fn in funcs:
            args += ["--dump", "%s=%s" % (fn, os.path.join(d, fn + ".bin"))]
        out = io.StringIO()
        with redirect_stdout(out), redirect_stderr(io.StringIO()):
            rc = ref_main(args)
        assert rc == 0
        dumps = {fn: open(os.path.join(d, fn + ".bin"), "rb").read()
                 for fn in funcs}
    return out.getvalue(), dumps


RUNS = [("acoustic_1d", cli_corpus.ACOUSTIC_1D, ("u",), 5, 0.1),
        ("acoustic_3d", cli_corpus.ACOUSTIC_3D, ("u", "rec"), 6, 1.0),
        ("snapshot_2d", cli_corpus.SNAPSHOT_2D, ("u", "us"), 10, 0.2),
        ("acoustic_3d_forced", cli_corpus.ACOUSTIC_3D_FORCED, ("u", "rec"), 6,
         1.0),
        ("acoustic_1d_forced", cli_corpus.ACOUSTIC_1D_FORCED, ("u", "rec"), 8,
         0.3),
        ("snapshot_2d_forced", cli_corpus.SNAPSHOT_2D_FORCED, ("u", "us"), 10,
         0.2)]


def main():
    out = {"corpus": [], "errors": [], "runs": {}}
    for text in cli_corpus.corpus():
        spec = parse_spec(text)
        out["corpus"].append({"sig": sig_sha(spec), "neq": len(spec.equations)})
    for text, _, _ in cli_corpus.ERRORS:
        try:
            parse_spec(text)
            raise AssertionError("no error for %r" % text)
        except SpecError as e:
            out["errors"].append([e.msg, e.line, e.col])
    for name, text, funcs, steps, dt in RUNS:
        stdout, dumps = run_dump(text, funcs, steps, dt)
        headers = {}
        arrays = {}
        for fn, raw in dumps.items():
            head, _, payload = raw.partition(b"\n")
            headers[fn] = head.decode()
            n, dtype, ndim, *ext = head.decode().split()
            arrays[fn] = np.frombuffer(
                payload, dtype="<f8" if dtype == "f64" else "<f4").reshape(
                tuple(int(e) for e in ext))
        np.savez_compressed(os.path.join(HERE, "arrays", "cli_" + name + ".npz"),
                            **arrays)
        out["runs"][name] = {"stdout": stdout, "headers": headers,
                             "sha": {fn: hashlib.sha256(raw).hexdigest()
                                     for fn, raw in dumps.items()}}
        print(name, stdout.strip().replace("\n", " | "))
    with open(os.path.join(HERE, "cli.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
