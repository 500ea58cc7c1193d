"""Batched device campaign (reference fault_lab/campaign.py) against the REAL
reference's records / ROC CSVs (tests/golden/make_golden*.py): identical runs,
faults and CSV formats; decisions equal wherever the reference's discrepancy
is clear of the thresholds (the clean-run rounding noise of two different FFT
implementations is not bit-identical, so values inside that band are only
compared approximately)."""

import csv
import io
import json
import math
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden")


def _read(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def _cases():
    spec = json.load(open(os.path.join(GOLD, "propagation.json")))["campaigns"]
    out = [("n64", dict(runs=40, inject_fraction=0.5, n=64, batch=4, precision="fp32", seed=3))]
    out += sorted(spec.items())
    return out


@pytest.mark.parametrize("name,kw", _cases(), ids=[c[0] for c in _cases()])
def test_campaign_matches_reference(name, kw):
    from paper_2405_02520_b200.fault_lab import (RECORD_COLUMNS, ROC_COLUMNS, CampaignConfig,
                                                 records_csv, roc_csv, run_campaign)
    kw = dict(kw)
    if "bits" in kw:
        kw["bits"] = tuple(kw["bits"])
    res = run_campaign(CampaignConfig(**kw))
    rec_text = records_csv(res)
    roc_text = roc_csv(res)
    assert rec_text.splitlines()[0] == ",".join(RECORD_COLUMNS)
    assert roc_text.splitlines()[0] == ",".join(ROC_COLUMNS)
    mine = list(csv.DictReader(io.StringIO(rec_text)))
    ref = _read(os.path.join(GOLD, f"campaign_{name}_records.csv"))
    assert len(mine) == len(ref) == kw["runs"]
    fp32 = kw["precision"] == "fp32"
    op_delta = 1e-4 if fp32 else 1e-9
    noise = 1e-5 if fp32 else 1e-12
    clean_ref = [float(r["discrepancy"]) for r in ref if r["injected"] == "0"]
    ref_dd = 10.0 * float(np.quantile(clean_ref, 0.999))
    assert res.default_delta == pytest.approx(ref_dd, rel=3.0)  # rounding-noise calibrated
    for m, r in zip(mine, ref):
        for k in ("run_id", "injected", "signal_idx", "element_idx", "bit"):
            assert m[k] == r[k], (name, r["run_id"], k)
        dm, dr = float(m["discrepancy"]), float(r["discrepancy"])
        if r["injected"] == "0":
            assert dm < 10 * max(clean_ref) + noise
            continue
        if math.isinf(dr):
            assert math.isinf(dm), (name, r["run_id"])
        elif dr > 10 * noise:
            assert dm == pytest.approx(dr, rel=5e-2), (name, r["run_id"])
        clear = lambda t: not (t / 3 < dr < 3 * t)  # noqa: E731
        if clear(ref_dd) and clear(res.default_delta):
            assert m["detected_at_default_delta"] == r["detected_at_default_delta"], (name, r["run_id"])
        if clear(op_delta) and (dr > 3 * op_delta or dr < noise):
            assert m["corrected"] == r["corrected"], (name, r["run_id"])
    # ROC: every rate within the share of reference runs whose discrepancy is
    # inside a factor 3 of that threshold
    roc_m = list(csv.DictReader(io.StringIO(roc_text)))
    roc_r = _read(os.path.join(GOLD, f"campaign_{name}_roc.csv"))
    disc_r = np.array([float(r["discrepancy"]) for r in ref])
    assert [row["delta"] for row in roc_m] == [row["delta"] for row in roc_r]
    n_inj = sum(r["injected"] == "1" for r in ref)
    n_clean = len(ref) - n_inj
    for a, b in zip(roc_m, roc_r):
        d = float(b["delta"])
        near = int(((disc_r > d / 3) & (disc_r < 3 * d)).sum())
        for k in ROC_COLUMNS[1:]:
            slack = near / max(min(n_inj, n_clean), 1) + 1e-12
            assert abs(float(a[k]) - float(b[k])) <= slack, (name, d, k)


def test_campaign_exponent_faults_all_detected_and_corrected():
    """Acceptance (test_acceptance.py:87-102 analogue): exponent-class flips
    of the output are all detected and corrected at the calibrated delta."""
    from paper_2405_02520_b200.fault_lab import CampaignConfig, run_campaign
    for prec, bits in (("fp32", tuple(range(25, 31))), ("fp64", tuple(range(57, 63)))):
        res = run_campaign(CampaignConfig(runs=200, inject_fraction=0.5, n=1 << 12, batch=16,
                                          precision=prec, seed=1, bits=bits))
        assert res.injected_count == 100
        assert res.detected_count == 100, prec
        assert res.corrected_count == 100, prec
        assert res.timing["protected_ms"] > 0
