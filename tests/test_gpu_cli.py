"""`transform` through the streamed native file path against the REAL
reference CLI's output files and printed reports (tests/golden/cli_transform.*),
plus the file path against the in-memory paths bit for bit (multi-chunk file,
injected fault, exit codes)."""

import contextlib
import io
import json
import os

import numpy as np
import pytest
import torch

from conftest import ROOT, rel_l2

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden")


def _run(argv):
    from paper_2405_02520_b200 import cli
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def test_cli_transform_matches_reference(tmp_path):
    cases = json.load(open(os.path.join(GOLD, "cli_transform.json")))
    arrays = np.load(os.path.join(GOLD, "cli_transform.npz"))
    for c in cases:
        x, ref = arrays[f"c{c['id']}_x"], arrays[f"c{c['id']}_y"]
        fi, fo = tmp_path / f"in{c['id']}.raw", tmp_path / f"out{c['id']}.raw"
        x.tofile(fi)
        argv = ["transform", "--input", str(fi), "--output", str(fo), "--n", str(c["n"]),
                "--precision", c["precision"], "--scheme", c["scheme"]] + (["--inverse"] if c["inverse"] else [])
        rc, out, _ = _run(argv)
        assert rc == c["rc"]
        mine, theirs = json.loads(out), json.loads(c["stdout"])
        assert mine == theirs, c["id"]
        y = np.fromfile(fo, dtype=x.dtype).reshape(x.shape)
        tol = (1e-5 if c["precision"] == "fp32" else 1e-12) * np.log2(c["n"])
        assert rel_l2(y, ref) < tol, c["id"]


def test_cli_transform_errors(tmp_path):
    bad = tmp_path / "bad.raw"
    bad.write_bytes(b"\0" * 24)
    rc, _, err = _run(["transform", "--input", str(bad), "--output", str(tmp_path / "o.raw"), "--n", "16"])
    assert rc == 1 and "input length mismatch: 24 bytes" in err
    assert not (tmp_path / "o.raw").exists()
    rc, _, err = _run(["transform", "--input", str(tmp_path / "missing.raw"), "--output",
                       str(tmp_path / "o.raw"), "--n", "16"])
    assert rc == 1


@pytest.mark.parametrize("n,prec,batch,scheme", [(2048, "fp32", 9000, "two_sided_group"),
                                                 (1 << 17, "fp64", 48, "one_sided"),
                                                 (512, "fp32", 64, "none")])
def test_file_stream_matches_device_path(tmp_path, n, prec, batch, scheme):
    """Multi-chunk file (several 32 MiB chunks), fault in the last chunk:
    output bytes and report equal the device-resident path's."""
    from paper_2405_02520_b200 import run_protected
    from paper_2405_02520_b200.abft import DetectionConfig
    from paper_2405_02520_b200.fault_lab import BitFlipInjector, FaultSpec
    from paper_2405_02520_b200.fft_core import build_twiddles, fit_group_size, make_plan
    from paper_2405_02520_b200.signal_io import transform_file
    dt = np.complex64 if prec == "fp32" else np.complex128
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))).astype(dt)
    fi, fo = tmp_path / "in.raw", tmp_path / "out.raw"
    x.tofile(fi)
    spec = FaultSpec(0, batch - 2, 7, "im", 30 if prec == "fp32" else 62)
    inj = BitFlipInjector(spec)
    rep, cnt, nb = transform_file(fi, fo, n, prec, scheme, injector=inj)
    assert nb == batch and inj.fired
    plan = fit_group_size(make_plan(n, prec, batch=batch), batch)
    cfg = DetectionConfig(delta=1e-4 if prec == "fp32" else 1e-9)
    yd, rd, cd = run_protected(plan, build_twiddles(plan), torch.from_numpy(x).cuda(), scheme, cfg,
                               injector=BitFlipInjector(spec))
    y = np.fromfile(fo, dtype=dt).reshape(batch, n)
    assert np.array_equal(y.view(np.uint8), yd.cpu().numpy().view(np.uint8))
    assert rep.to_json() == rd.to_json() and cnt.total == cd.total
    if scheme != "none":
        assert [c["signal"] for c in rep.corrected] == [batch - 2]


def test_cli_inject_and_bench(tmp_path):
    """`inject` writes the reference's ROC / records CSV formats and prints the
    summary JSON; `bench` emits the reference's CSV columns."""
    roc, rec = tmp_path / "roc.csv", tmp_path / "records.csv"
    rc, out, _ = _run(["inject", "--runs", "40", "--n", "64", "--batch", "4", "--seed", "3",
                       "--roc-out", str(roc), "--records-out", str(rec)])
    assert rc == 0
    summary = json.loads(out)
    assert set(summary) == {"runs", "injected", "detected_at_default_delta", "corrected",
                            "default_delta", "recompute_count"}
    assert summary["runs"] == 40 and summary["injected"] == 20
    gold = open(os.path.join(GOLD, "campaign_n64_records.csv")).read().splitlines()
    mine = rec.read_text().splitlines()
    assert mine[0] == gold[0] and len(mine) == len(gold)
    # run ids, injection flags and fault coordinates are the reference's
    assert [l.split(",")[:5] for l in mine] == [l.split(",")[:5] for l in gold]
    assert roc.read_text().splitlines()[0] == open(os.path.join(GOLD, "campaign_n64_roc.csv")).read().splitlines()[0]
    out_csv = tmp_path / "bench.csv"
    rc, _, _ = _run(["bench", "--n-list", "64", "--batch-list", "16", "--trials", "2", "--out", str(out_csv)])
    assert rc == 0
    lines = out_csv.read_text().splitlines()
    assert lines[0] == "n,batch,scheme,backend,trials,mean_s,stdev_s,pass_count,recompute_count"
    assert len(lines) == 1 + 3  # none / one_sided / two_sided_group x backend cuda
