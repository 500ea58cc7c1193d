"""Throughput sweep over sizes (both precisions): fused ABFT-on vs off and
cuFFT (torch.fft, comparison only), per-pass HBM GB/s against the measured
copy peak. Prints one JSON object per size; writes gpurun_out/sweep.json.

    python tools/sweep.py [--sizes 3-25] [--prec fp32,fp64] [--gib 1]
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
    ap.add_argument("--sizes", default="3-25")
    ap.add_argument("--prec", default="fp32,fp64")
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-cufft", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    args = ap.parse_args()
    import torch

    from paper_2405_02520_b200 import _lib, make_plan
    from paper_2405_02520_b200.abft import make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    lo, hi = (int(v) for v in args.sizes.split("-"))
    out = []
    for prec in args.prec.split(","):
        dt = torch.complex64 if prec == "fp32" else torch.complex128
        es = 8 if prec == "fp32" else 16
        total = int(args.gib * (1 << 30)) // es
        x = torch.randn(total, dtype=dt, device="cuda")
        y = torch.empty_like(x)
        for logn in range(lo, hi + 1):
            n = 1 << logn
            b = total // n
            if b < 1:
                continue
            plan = fit_group_size(make_plan(n, prec, batch=b), b)
            h = native_plan(plan, 0)
            row = make_encoding("wang", n).device_row(dt)
            rep = _lib.Report()
            delta = 1e-4 if prec == "fp32" else 1e-9

            def on():
                _lib.check(lib.tfft_protect_launch(h.handle, x.data_ptr(), y.data_ptr(), b, 3, delta,
                                                   0.0, row.data_ptr(), None, None, 0,
                                                   ctypes.byref(rep), sp))

            def off():
                _lib.check(lib.tfft_execute(h.handle, x.data_ptr(), y.data_ptr(), b, 0, sp))

            def cufft():
                torch.fft.fft(x[: b * n].view(b, n), out=y[: b * n].view(b, n))

            def timed(fn):
                for _ in range(2):
                    fn()
                ts = []
                for _ in range(args.reps):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                return float(np.median(ts))

            t_on, t_off = timed(on), timed(off)
            t_cu = None if args.no_cufft else timed(cufft)
            passes = lib.tfft_plan_exec_passes(h.handle)  # HBM passes actually launched
            byts = 2.0 * b * n * es
            r = dict(prec=prec, n=n, batch=b, passes=passes, api_stages=len(plan.stages), ms_on=round(t_on, 4),
                     ms_off=round(t_off, 4), ms_cufft=None if t_cu is None else round(t_cu, 4),
                     gbs_pass_on=round(passes * byts / t_on / 1e6, 1),
                     frac_pass_on=round(passes * byts / t_on / 1e6 / peak, 4),
                     gbs_pass_off=round(passes * byts / t_off / 1e6, 1),
                     gflops_on=round(5 * n * math.log2(n) * b / t_on / 1e6, 1),
                     abft_overhead_pct=round(100 * (t_on / t_off - 1), 2),
                     vs_cufft_on=None if t_cu is None else round(t_cu / t_on, 3),
                     flagged=int(rep.n_flagged))
            out.append(r)
            print(json.dumps(r), flush=True)
        del x, y
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
