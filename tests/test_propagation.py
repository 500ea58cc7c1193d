"""propagation_footprint (reference fault_lab/propagation.py) against the
footprints the real reference printed (tests/golden/make_golden_campaign.py);
host utility, no GPU."""

import json
import os

import pytest

from conftest import ROOT


def test_footprints_match_reference():
    from paper_2405_02520_b200.fault_lab import propagation_footprint
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "propagation.json")))["footprints"]
    assert gold
    for g in gold:
        assert propagation_footprint(g["n"], g["stage"], element=g["element"]) == g["footprint"], g


def test_footprint_doubles_per_remaining_step_and_validates():
    from paper_2405_02520_b200.fault_lab import propagation_footprint
    n = 256
    steps = 8
    for s in range(steps + 1):
        assert propagation_footprint(n, s) == 2 ** (steps - s)
    with pytest.raises(ValueError):
        propagation_footprint(12, 0)
    with pytest.raises(ValueError):
        propagation_footprint(16, 5)
    with pytest.raises(ValueError):
        propagation_footprint(16, 1, element=16)
