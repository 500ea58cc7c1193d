"""Golden fixtures for the campaign and propagation rows, produced by the REAL
reference (build container only; see make_golden.py for the mechanics):

    python tests/golden/make_golden_campaign.py

Writes campaign_*.csv (records + ROC of small campaigns in both precisions,
with the output / input / stage hooks) and propagation.json (footprints)."""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import _reference  # noqa: E402

CAMPAIGNS = {
    # name: CampaignConfig kwargs
    "fp64_n256_output": dict(runs=40, inject_fraction=0.5, n=256, batch=4, precision="fp64", seed=5),
    "fp32_n512_input": dict(runs=30, inject_fraction=0.5, n=512, batch=8, precision="fp32", seed=9,
                            stage="input", bits=(23, 24, 25, 26, 27, 28, 29, 30)),
    "fp32_n16384_stage0": dict(runs=12, inject_fraction=0.5, n=16384, batch=2, precision="fp32", seed=11,
                               stage="stage:0", bits=(27, 28, 29, 30)),
    "fp64_n64_onesided": dict(runs=24, inject_fraction=0.5, n=64, batch=4, precision="fp64", seed=13,
                              scheme="one_sided", bits=(55, 56, 57, 58, 59, 60, 61, 62)),
}

FOOTPRINTS = [(8, s, 3) for s in range(4)] + [(64, s, 17) for s in range(7)] + [(1024, s, 511) for s in (0, 3, 7, 10)]


def main():
    _reference(None)
    from fftshield.fault_lab import CampaignConfig, propagation_footprint, records_csv, roc_csv, run_campaign
    for name, kw in CAMPAIGNS.items():
        res = run_campaign(CampaignConfig(**kw))
        with open(os.path.join(HERE, f"campaign_{name}_records.csv"), "w") as f:
            f.write(records_csv(res))
        with open(os.path.join(HERE, f"campaign_{name}_roc.csv"), "w") as f:
            f.write(roc_csv(res))
        print(name, res.default_delta, res.injected_count, res.detected_count, res.corrected_count,
              res.recompute_count)
    fp = [dict(n=n, stage=s, element=e, footprint=propagation_footprint(n, s, element=e)) for n, s, e in FOOTPRINTS]
    with open(os.path.join(HERE, "propagation.json"), "w") as f:
        json.dump(dict(campaigns=CAMPAIGNS, footprints=fp), f, indent=1)


if __name__ == "__main__":
    main()
