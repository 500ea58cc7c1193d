"""Golden C4 campaigns produced by the REAL reference (build container only):

    python tests/golden/make_golden_c4.py [name ...]

SURVEY §8(d) C4 = ``run_campaign(CampaignConfig(runs=2000, inject_fraction=0.5,
n=2**16, batch=16, precision=p, seed=1))`` for fp32 and fp64, plus the
exponent-class variants (bits 25-30 fp32, the reference acceptance's class,
tests/test_acceptance.py:97; bits 57-62 the fp64 analogue). Each campaign runs
the reference's own ``run_campaign`` unmodified, one process per campaign, and
writes ``c4_<name>_records.csv`` / ``c4_<name>_roc.csv`` (the reference's CSV
formats) plus a summary line in ``c4_summary.json``. About 7-12 min per
campaign on one core.
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

C4 = {
    "fp32": dict(precision="fp32"),
    "fp64": dict(precision="fp64"),
    "fp32_exp": dict(precision="fp32", bits=(25, 26, 27, 28, 29, 30)),
    "fp64_exp": dict(precision="fp64", bits=(57, 58, 59, 60, 61, 62)),
}
BASE = dict(runs=2000, inject_fraction=0.5, n=2**16, batch=16, seed=1)


def _one(name):
    from make_golden import _reference
    _reference(None)
    from fftshield.fault_lab import CampaignConfig, records_csv, roc_csv, run_campaign
    t0 = time.perf_counter()
    res = run_campaign(CampaignConfig(**BASE, **C4[name]))
    dt = time.perf_counter() - t0
    with open(os.path.join(HERE, f"c4_{name}_records.csv"), "w") as f:
        f.write(records_csv(res))
    with open(os.path.join(HERE, f"c4_{name}_roc.csv"), "w") as f:
        f.write(roc_csv(res))
    return name, dict(default_delta=res.default_delta, injected=res.injected_count,
                      detected=res.detected_count, corrected=res.corrected_count,
                      recompute=res.recompute_count, seconds=round(dt, 1))


def main():
    names = sys.argv[1:] or list(C4)
    from make_golden import _reference
    _reference(None)  # build the scratch copy once, before the workers start
    with mp.get_context("fork").Pool(len(names)) as pool:
        out = dict(pool.map(_one, names))
    path = os.path.join(HERE, "c4_summary.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(out)
    with open(path, "w") as f:
        json.dump({"config": BASE, "variants": C4, **old}, f, indent=1, default=list)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
