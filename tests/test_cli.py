"""CLI on the B200 backend: the spec parser builds
the same equation trees as the reference's (signature parity over a
corpus, same diagnostics), and `run --dump` on the GPU reproduces the
reference CLI's dumps bit for bit (goldens: tests/golden/make_golden_cli.py,
run against the real reference)."""

import hashlib
import json
import os

import numpy as np
import pytest

import cli_corpus
from paper_1807_03032_b200.cli import main, parse_spec, pretty_print, report_text
from paper_1807_03032_b200.cli.spec import SpecError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden():
    with open(os.path.join(GOLD, "cli.json")) as f:
        return json.load(f)


def _sig(spec):
    return hashlib.sha256(repr(spec.signature()).encode()).hexdigest()


def test_corpus_signatures_match_reference_parser():
    gold = _golden()["corpus"]
    texts = cli_corpus.corpus()
    assert len(texts) == len(gold)
    for text, g in zip(texts, gold):
        spec = parse_spec(text)
        assert len(spec.equations) == g["neq"], text
        assert _sig(spec) == g["sig"], text


def test_diagnostics_match_reference():
    for (text, frag, line), g in zip(cli_corpus.ERRORS, _golden()["errors"]):
        with pytest.raises(SpecError) as err:
            parse_spec(text)
        assert frag in err.value.msg and err.value.line == line
        assert [err.value.msg, err.value.line, err.value.col] == g, text


def test_pretty_print_round_trip():
    for text in cli_corpus.corpus():
        spec = parse_spec(text)
        assert parse_spec(pretty_print(spec)).signature() == spec.signature()


def test_parse_details():
    spec = parse_spec(cli_corpus.ACOUSTIC_1D)
    assert len(spec.functions) == 3 and len(spec.statements) == 2
    assert len(spec.equations) == 3
    assert spec.params == {"steps": 10, "mode": "advanced", "precision": "f64"}
    snap = parse_spec(cli_corpus.SNAPSHOT_2D).functions["us"]
    assert snap.time_dim.kind == "conditional" and snap.time_dim.factor == 3
    spec = parse_spec("grid shape=(21,)\ntimefunction u\n"
                      "sparsetimefunction rec npoint=2 coords=((5.0,), (9.5,))\n"
                      "rec.interpolate(u)\n")
    assert spec.functions["rec"].coordinate_values == [(5.0,), (9.5,)]


def _write(tmp_path, text):
    p = tmp_path / "problem.spec"
    p.write_text(text)
    return str(p)


def test_compile_and_plan(tmp_path, capsys):
    path = _write(tmp_path, cli_corpus.ACOUSTIC_1D)
    plan = tmp_path / "plan.txt"
    assert main(["compile", path, "--emit-plan", str(plan)]) == 0
    assert "compiled 3 equations into" in capsys.readouterr().out
    assert "cluster 0" in plan.read_text()


def test_report_deterministic_and_ordered():
    spec = parse_spec(cli_corpus.ACOUSTIC_1D)
    a = report_text(spec, "aggressive")
    assert a == report_text(parse_spec(cli_corpus.ACOUSTIC_1D), "aggressive")
    tot = {m: int([ln for ln in report_text(parse_spec(cli_corpus.ACOUSTIC_1D),
                                           m).splitlines()
                   if ln.startswith("total after:")][0].split(":")[1])
           for m in ("basic", "aggressive")}
    assert tot["aggressive"] <= tot["basic"]


def test_error_exit_code(tmp_path, capsys):
    path = _write(tmp_path, "grid shape=(11,)\neq u = 1\n")
    assert main(["compile", path]) == 1
    err = capsys.readouterr().err
    assert "undeclared identifier" in err and "line 2" in err


RUNS = [("acoustic_1d", cli_corpus.ACOUSTIC_1D, ("u",), 5, 0.1),
        ("acoustic_3d", cli_corpus.ACOUSTIC_3D, ("u", "rec"), 6, 1.0),
        ("snapshot_2d", cli_corpus.SNAPSHOT_2D, ("u", "us"), 10, 0.2),
        ("acoustic_3d_forced", cli_corpus.ACOUSTIC_3D_FORCED, ("u", "rec"), 6,
         1.0),
        ("acoustic_1d_forced", cli_corpus.ACOUSTIC_1D_FORCED, ("u", "rec"), 8,
         0.3),
        ("snapshot_2d_forced", cli_corpus.SNAPSHOT_2D_FORCED, ("u", "us"), 10,
         0.2)]


@pytest.mark.gpu
@pytest.mark.parametrize("row", RUNS, ids=[r[0] for r in RUNS])
def test_run_dump_bitwise_vs_reference_cli(row, tmp_path, capsys):
    name, text, funcs, steps, dt = row
    gold = _golden()["runs"][name]
    path = _write(tmp_path, text)
    args = ["run", path, "--steps", str(steps), "--dt", repr(dt)]
    for fn in funcs:
        args += ["--dump", "%s=%s" % (fn, tmp_path / (fn + ".bin"))]
    assert main(args) == 0
    assert capsys.readouterr().out == gold["stdout"]
    ref = np.load(os.path.join(GOLD, "arrays", "cli_%s.npz" % name))
    for fn in funcs:
        raw = (tmp_path / (fn + ".bin")).read_bytes()
        head, _, payload = raw.partition(b"\n")
        assert head.decode() == gold["headers"][fn]
        if name.endswith("_forced"):
            # finite, non-zero data: the dump must be the reference's bytes
            got = np.frombuffer(payload, dtype=ref[fn].dtype)
            assert np.isfinite(got).all() and np.count_nonzero(got) > 0
            assert hashlib.sha256(raw).hexdigest() == gold["sha"][fn], fn
            continue
        if hashlib.sha256(raw).hexdigest() != gold["sha"][fn]:
            # the specs leave m zero (the CLI cannot set data), so the
            # wavefields hold inf/NaN; NaN payload bits carry no meaning:
            # same NaN positions, every other value bit for bit
            got = np.frombuffer(payload, dtype=ref[fn].dtype).reshape(ref[fn].shape)
            nan_g, nan_r = np.isnan(got), np.isnan(ref[fn])
            assert np.array_equal(nan_g, nan_r), fn
            ui = np.uint32 if got.dtype == np.float32 else np.uint64
            bad = np.argwhere((got.view(ui) != ref[fn].view(ui)) & ~nan_r)
            assert len(bad) == 0, (fn, len(bad), bad[:3])
