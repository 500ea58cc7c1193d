"""Golden fixtures for the campaign, propagation, CLI and descriptor rows,
produced by the REAL reference (build container only; see make_golden.py for
the mechanics):

    python tests/golden/make_golden_campaign.py

Writes campaign_*.csv (records + ROC of small campaigns in both precisions,
with the output / input / stage hooks), propagation.json (footprints),
descriptors.json (`fftshield plan` JSON) and cli_transform.npz/json (raw files
transformed by `fftshield transform`, with the printed reports)."""

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
    # ---- `fftshield plan` descriptors
    from fftshield import planner
    desc = []
    for n in (2, 8, 64, 1024, 2**13, 2**17, 2**20, 2**23, 2**25):
        for b in (1, 16, 64):
            for mode in planner.FT_MODES:
                d = planner.emit_descriptor(planner.select_parameters(n, b), mode)
                desc.append(dict(n=n, batch=b, ft_mode=mode, json=planner.render_descriptor(d)))
    with open(os.path.join(HERE, "descriptors.json"), "w") as f:
        json.dump(desc, f)
    # ---- `fftshield transform` on raw files
    import io
    import contextlib
    import tempfile
    import numpy as np
    from fftshield import cli
    cases, arrays = [], {}
    for i, (n, b, prec, scheme, inverse) in enumerate([(256, 16, "fp32", "two_sided_group", False),
                                                       (1024, 8, "fp64", "one_sided", True),
                                                       (2**14, 4, "fp32", "none", False)]):
        rng = np.random.default_rng([4242, i])
        x = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(
            np.complex64 if prec == "fp32" else np.complex128)
        with tempfile.TemporaryDirectory() as td:
            fi, fo = os.path.join(td, "in.raw"), os.path.join(td, "out.raw")
            x.tofile(fi)
            argv = ["transform", "--input", fi, "--output", fo, "--n", str(n), "--precision", prec,
                    "--scheme", scheme] + (["--inverse"] if inverse else [])
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = cli.main(argv)
            y = np.fromfile(fo, dtype=x.dtype).reshape(b, n)
        arrays[f"c{i}_x"], arrays[f"c{i}_y"] = x, y
        cases.append(dict(id=i, n=n, batch=b, precision=prec, scheme=scheme, inverse=inverse, rc=rc,
                          stdout=buf.getvalue()))
    np.savez_compressed(os.path.join(HERE, "cli_transform.npz"), **arrays)
    with open(os.path.join(HERE, "cli_transform.json"), "w") as f:
        json.dump(cases, f, indent=1)
    # ---- element-level two-sided tiles (abft/element.py)
    from fftshield.abft import DetectionConfig, UnrecoverableError, make_encoding, two_sided_element
    el_cases, el_arrays = [], {}
    specs = [  # (r, B, row enc, col enc, delta, abs_floor, edits [(i, j, kind, value)])
        (8, 8, "ones", "linear", 1e-6, 1e-12, []),
        (4, 4, "ones", "linear", 1e-6, 1e-12, [(3, 2, "add", 7.0)]),
        (16, 5, "wang", "linear", 1e-9, 1e-12, [(5, 1, "add", 3.0 - 2.0j)]),
        (8, 6, "wang", "ones", 1e-9, 1e-12, [(2, 3, "set", complex(np.inf, 0.0))]),
        (8, 8, "ones", "linear", 1e-6, 1e-12, [(1, 1, "add", 5.0), (2, 6, "add", 4.0)]),
        (8, 8, "ones", "linear", 1e-6, 1e-12, [(1, 3, "add", 5.0), (6, 3, "add", -2.0j)]),
        (32, 32, "wang", "wang", 1e-9, 1e-12, [(31, 0, "add", 1e-3)]),
        (2, 3, "linear", "linear", 1e-6, 0.0, [(0, 2, "add", 1.0)]),
    ]
    for cid, (r, b, er, ec, delta, floor, edits) in enumerate(specs):
        rng = np.random.default_rng([99, cid])
        x = rng.standard_normal((r, b)) + 1j * rng.standard_normal((r, b))

        def inject(y, _e=edits):
            for i, j, kind, val in _e:
                if kind == "add":
                    y[i, j] += val
                else:
                    y[i, j] = val

        try:
            y, rep = two_sided_element(r, x, make_encoding(er, r), make_encoding(ec, b),
                                       DetectionConfig(delta=delta, abs_floor=floor),
                                       inject=inject if edits else None)
            outcome = dict(error=None, located=list(rep.located) if rep.located else None,
                           corrected=rep.corrected)
            el_arrays[f"e{cid}_y"] = y
            el_arrays[f"e{cid}_rel"] = rep.col_discrepancies
        except UnrecoverableError as exc:
            outcome = dict(error=str(exc), located=None, corrected=False)
        el_arrays[f"e{cid}_x"] = x
        el_cases.append(dict(id=cid, r=r, b=b, enc_row=er, enc_col=ec, delta=delta, abs_floor=floor,
                             edits=[[i, j, k, [complex(v).real, complex(v).imag]] for i, j, k, v in edits],
                             **outcome))
    np.savez_compressed(os.path.join(HERE, "element.npz"), **el_arrays)
    with open(os.path.join(HERE, "element.json"), "w") as f:
        json.dump(el_cases, f, indent=1)
    fp = [dict(n=n, stage=s, element=e, footprint=propagation_footprint(n, s, element=e)) for n, s, e in FOOTPRINTS]
    with open(os.path.join(HERE, "propagation.json"), "w") as f:
        json.dump(dict(campaigns=CAMPAIGNS, footprints=fp), f, indent=1)


if __name__ == "__main__":
    main()
