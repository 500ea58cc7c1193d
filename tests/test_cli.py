"""CLI / file-format / descriptor parity that needs no GPU: `plan` JSON is
byte-identical to the reference's (tests/golden/descriptors.json), raw file
helpers follow signal_io.py, usage errors exit 1."""

import contextlib
import io
import json
import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")


def _run(argv):
    from paper_2405_02520_b200 import cli
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def test_descriptors_byte_identical_to_reference():
    from paper_2405_02520_b200 import planner
    gold = json.load(open(os.path.join(GOLD, "descriptors.json")))
    assert len(gold) > 50
    for g in gold:
        d = planner.emit_descriptor(planner.select_parameters(g["n"], g["batch"]), g["ft_mode"])
        assert planner.render_descriptor(d) == g["json"], (g["n"], g["batch"], g["ft_mode"])
    with pytest.raises(ValueError):
        planner.emit_descriptor(planner.select_parameters(64), "bogus")


def test_cli_plan_and_propagate():
    gold = {(g["n"], g["batch"], g["ft_mode"]): g["json"]
            for g in json.load(open(os.path.join(GOLD, "descriptors.json")))}
    rc, out, _ = _run(["plan", "--n", "1024", "--batch", "16", "--ft-mode", "two_sided"])
    assert rc == 0 and out == gold[(1024, 16, "two_sided")] + "\n"
    rc, out, _ = _run(["propagate", "--n", "64", "--stage", "3", "--element", "5"])
    assert rc == 0 and json.loads(out) == {"corrupted_outputs": 8, "element": 5, "inject_stage": 3, "n": 64}


def test_cli_usage_errors_exit_1(tmp_path):
    assert _run(["bogus"])[0] == 1
    assert _run(["plan", "--n", "12"])[0] == 1
    rc, _, err = _run(["propagate", "--n", "16", "--stage", "9"])
    assert rc == 1 and "inject_stage" in err
    bad = tmp_path / "bad.raw"
    bad.write_bytes(b"\0" * 12)
    from paper_2405_02520_b200 import signal_io
    with pytest.raises(ValueError, match="input length mismatch: 12 bytes"):
        signal_io.signal_count(bad, 4, "fp32")


def test_signal_files_round_trip(tmp_path):
    from paper_2405_02520_b200 import signal_io
    rng = np.random.default_rng(1)
    for prec, dt in (("fp32", np.complex64), ("fp64", np.complex128)):
        x = (rng.standard_normal((3, 16)) + 1j * rng.standard_normal((3, 16))).astype(dt)
        f = tmp_path / f"s_{prec}.raw"
        signal_io.write_signals(f, x, prec)
        assert f.stat().st_size == x.size * 2 * (4 if prec == "fp32" else 8)
        # interleaved little-endian (re, im) pairs
        raw = np.fromfile(f, dtype="<f4" if prec == "fp32" else "<f8")
        assert np.array_equal(raw[0::2], x.real.ravel()) and np.array_equal(raw[1::2], x.imag.ravel())
        y = signal_io.read_signals(f, 16, prec)
        assert y.dtype == dt and y.shape == (3, 16) and np.array_equal(x, y)
        assert signal_io.signal_count(f, 16, prec) == 3
        with pytest.raises(ValueError, match="input length mismatch"):
            signal_io.read_signals(f, 32 if prec == "fp32" else 7 * 16, prec)
