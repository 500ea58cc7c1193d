"""On-GPU tuner for the single-kernel launch variants (codegen.SINGLE_CANDIDATES).

For every (precision, log2 N) it checks each compiled variant against an
fp64 numpy FFT on a small batch, then times it on a 1 GiB batch with ABFT on
(two_sided_group, fused) and off, and writes the results to
gpurun_out/tune_single.json. The winners go into codegen.SINGLE_CHOICE.

    python tools/tune.py [--sizes 3-13] [--prec fp32,fp64] [--reps 5]

Needs the tuning build (every candidate compiled):
    TFFT_TUNE=1 python -m paper_2405_02520_b200.build
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1-13")
    ap.add_argument("--prec", default="fp32,fp64")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--delta", type=float, default=None,
                    help="detection threshold of the timed ABFT launches (default 1e-2 fp32 / 1e-9 "
                         "fp64: no clean-data false alarms, so the timing is the fused kernel's)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "tune_single.json"))
    args = ap.parse_args()
    import torch

    from paper_2405_02520_b200 import _lib, make_plan
    from paper_2405_02520_b200.abft import make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan

    lo, hi = (int(v) for v in args.sizes.split("-"))
    lib = _lib.load()
    sp = torch.cuda.current_stream().cuda_stream
    results = []
    for prec in args.prec.split(","):
        pc = _lib.FP32 if prec == "fp32" else _lib.FP64
        dt = torch.complex64 if prec == "fp32" else torch.complex128
        esize = 8 if prec == "fp32" else 16
        total = int(args.gib * (1 << 30)) // esize
        x = torch.randn(total, dtype=dt, device="cuda")
        y = torch.empty_like(x)
        for logn in range(lo, hi + 1):
            n = 1 << logn
            b = total // n
            plan = fit_group_size(make_plan(n, prec, batch=b), b)
            h = native_plan(plan, 0)
            row = make_encoding("wang", n).device_row(dt)
            rep = _lib.Report()
            cap = 64
            fl = (_lib.Flag * cap)()
            i64 = (ctypes.c_int64 * cap)
            cg, cs, ur = i64(), i64(), i64()
            rep.flagged, rep.flagged_cap = fl, cap
            rep.corrected_group, rep.corrected_signal, rep.corrected_cap = cg, cs, cap
            rep.unrecoverable, rep.unrecoverable_cap = ur, cap
            small = torch.randn(64, n, dtype=dt, device="cuda")
            ref = np.fft.fft(small.cpu().numpy().astype(np.complex128), axis=-1)
            delta = args.delta if args.delta is not None else (1e-2 if prec == "fp32" else 1e-9)
            from paper_2405_02520_b200 import codegen
            ncand = len(codegen.SINGLE_CANDIDATES[prec][logn])
            for v in range(ncand):
                if lib.tfft_tune_select(pc, logn, v) != 0:
                    continue  # not compiled in this (size-restricted) tuning build
                out = torch.empty_like(small)
                _lib.check(lib.tfft_execute(h.handle, small.data_ptr(), out.data_ptr(), 64, 0, sp))
                got = out.cpu().numpy().astype(np.complex128)
                err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))

                def run_off():
                    _lib.check(lib.tfft_execute(h.handle, x.data_ptr(), y.data_ptr(), b, 0, sp))

                def run_on():
                    _lib.check(lib.tfft_protect_launch(h.handle, x.data_ptr(), y.data_ptr(), b, 3,
                                                       delta, 0.0,
                                                       row.data_ptr(), None, None, 0,
                                                       ctypes.byref(rep), sp))

                def timed(fn):
                    for _ in range(2):
                        fn()
                    ts = []
                    for _ in range(args.reps):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                        fn()
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    return float(np.median(ts))

                t_off = timed(run_off)
                t_on = timed(run_on)
                gbs = 2 * b * n * esize / t_on / 1e6
                r = dict(prec=prec, logn=logn, variant=v, err=err, ms_off=t_off, ms_on=t_on,
                         gbs_on=gbs, gbs_off=2 * b * n * esize / t_off / 1e6)
                results.append(r)
                print(json.dumps(r), flush=True)
            _lib.check(lib.tfft_tune_select(pc, logn, -1))
        del x, y
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(results, f, indent=1)
    best = {}
    for r in results:
        tol = 1e-6 * r["logn"] if r["prec"] == "fp32" else 1e-14 * r["logn"]
        if r["err"] > tol:
            print("BROKEN", r)
            continue
        k = (r["prec"], r["logn"])
        if k not in best or r["ms_on"] < best[k]["ms_on"]:
            best[k] = r
    print("BEST", json.dumps({f"{p}:{l}": [v["variant"], round(v["gbs_on"], 1)]
                              for (p, l), v in sorted(best.items())}))


if __name__ == "__main__":
    main()
