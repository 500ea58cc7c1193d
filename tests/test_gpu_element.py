"""Element-level two-sided ABFT (reference abft/element.py) on the device
against the REAL reference's outcomes on the same tiles and injections
(tests/golden/element.*): same located (row, col), same corrected / error,
outputs and column discrepancies within fp64 tolerance."""

import json
import os

import numpy as np
import pytest

from conftest import ROOT, rel_l2

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden")


def test_element_tiles_match_reference():
    from paper_2405_02520_b200.abft import (DetectionConfig, UnrecoverableError, make_encoding,
                                            two_sided_element)
    cases = json.load(open(os.path.join(GOLD, "element.json")))
    arrays = np.load(os.path.join(GOLD, "element.npz"))
    for c in cases:
        x = arrays[f"e{c['id']}_x"]
        edits = [(i, j, k, complex(v[0], v[1])) for i, j, k, v in c["edits"]]

        def inject(y, _e=edits):
            for i, j, kind, val in _e:
                if kind == "add":
                    y[i, j] += val
                else:
                    y[i, j] = val

        cfg = DetectionConfig(delta=c["delta"], abs_floor=c["abs_floor"])
        args = (c["r"], x, make_encoding(c["enc_row"], c["r"]), make_encoding(c["enc_col"], c["b"]), cfg)
        kw = dict(inject=inject if edits else None)
        if c["error"]:
            with pytest.raises(UnrecoverableError, match=c["error"]):
                two_sided_element(*args, **kw)
            continue
        y, rep = two_sided_element(*args, **kw)
        assert rep.corrected == c["corrected"], c["id"]
        assert (list(rep.located) if rep.located else None) == c["located"], c["id"]
        assert rel_l2(y, arrays[f"e{c['id']}_y"]) < 1e-12, c["id"]
        ref_rel = arrays[f"e{c['id']}_rel"]
        fin = np.isfinite(ref_rel)
        assert np.array_equal(fin, np.isfinite(rep.col_discrepancies))
        big = fin & (ref_rel > 1e-6)
        assert np.allclose(rep.col_discrepancies[big], ref_rel[big], rtol=1e-6)


def test_element_fault_free_and_validation():
    from paper_2405_02520_b200.abft import DetectionConfig, make_encoding, two_sided_element
    rng = np.random.default_rng(3)
    tile = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
    y, rep = two_sided_element(8, tile, make_encoding("ones", 8), make_encoding("linear", 8),
                               DetectionConfig(delta=1e-6, abs_floor=1e-12))
    assert rep.located is None and not rep.corrected
    w = np.exp(-2j * np.pi * np.outer(np.arange(8), np.arange(8)) / 8)
    np.testing.assert_allclose(y, w @ tile, atol=1e-9)
    with pytest.raises(ValueError):
        two_sided_element(3, tile[:3], make_encoding("ones", 3), make_encoding("ones", 8),
                          DetectionConfig(delta=1e-6))
    with pytest.raises(ValueError):
        two_sided_element(8, tile[:4], make_encoding("ones", 8), make_encoding("ones", 8),
                          DetectionConfig(delta=1e-6))
