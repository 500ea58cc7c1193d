"""On-GPU tuner for the multi-pass stage kernels (codegen.PASS_CANDIDATES).

Walks N = 2^14 .. 2^25 (reference plans), and for every (precision, stage dim
L, stage kind) not tuned yet, times the whole protected transform (ABFT on,
1 GiB batch) with each compiled variant of that stage, keeping the other
stages at their current best. Correctness of every variant is checked against
numpy on a small batch. Prints PASS_CHOICE for codegen.py and writes
gpurun_out/tune_pass.json.

Needs the tuning build (every candidate compiled):
    TFFT_TUNE=1 python -m paper_2405_02520_b200.build
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="fp32,fp64")
    ap.add_argument("--sizes", default="14-25")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "tune_pass.json"))
    args = ap.parse_args()
    import torch

    from paper_2405_02520_b200 import _lib, make_plan
    from paper_2405_02520_b200.abft import make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan

    lib = _lib.load()
    sp = torch.cuda.current_stream().cuda_stream
    lo, hi = (int(v) for v in args.sizes.split("-"))
    results, choice = [], {}
    for prec in args.prec.split(","):
        pc = _lib.FP32 if prec == "fp32" else _lib.FP64
        dt = torch.complex64 if prec == "fp32" else torch.complex128
        es = 8 if prec == "fp32" else 16
        total = int(args.gib * (1 << 30)) // es
        x = torch.randn(total, dtype=dt, device="cuda")
        y = torch.empty_like(x)
        best = {}  # (logl, kind) -> variant
        for logn in range(lo, hi + 1):
            n = 1 << logn
            b = max(1, total // n)
            plan = fit_group_size(make_plan(n, prec, batch=b), b)
            h = native_plan(plan, 0)
            row = make_encoding("wang", n).device_row(dt)
            rep = _lib.Report()
            nst = len(plan.stages)
            small = torch.randn(2, n, dtype=dt, device="cuda")
            ref = np.fft.fft(small.cpu().numpy().astype(np.complex128), axis=-1)
            dims = list(plan.dims)
            if lib.tfft_plan_exec_passes(h.handle) == 3 and nst == 2:
                # executed as the library's balanced 3-pass split (larger parts last)
                q, r3 = divmod(logn, 3)
                dims = [1 << (q + (1 if i >= 3 - r3 else 0)) for i in range(3)]
                nst = 3
            for k, d in enumerate(dims):
                logl = d.bit_length() - 1
                kind = 0 if k == 0 else (2 if k == nst - 1 else 1)
                if (logl, kind) in best:
                    continue
                from paper_2405_02520_b200 import codegen
                ncand = len(codegen.PASS_CANDIDATES[prec].get(logl, []))
                timings = []
                for v in range(ncand):
                    if lib.tfft_tune_pass_select(pc, logl, kind, v) != 0:
                        continue  # not compiled in this build
                    out = torch.empty_like(small)
                    try:
                        _lib.check(lib.tfft_execute(h.handle, small.data_ptr(), out.data_ptr(), 2, 0, sp))
                    except NotImplementedError:
                        continue  # tile too wide for this split
                    err = float(np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref))

                    def on():
                        _lib.check(lib.tfft_protect_launch(h.handle, x.data_ptr(), y.data_ptr(), b, 3,
                                                           1e-4 if prec == "fp32" else 1e-9, 0.0,
                                                           row.data_ptr(), None, None, 0,
                                                           ctypes.byref(rep), sp))
                    for _ in range(2):
                        on()
                    ts = []
                    for _ in range(args.reps):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                        on()
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    ms = float(np.median(ts))
                    ok = err <= (1e-6 if prec == "fp32" else 1e-14) * logn
                    r = dict(prec=prec, n=n, logl=logl, kind=kind, variant=v, ms=ms, err=err, ok=ok,
                             gbs_pass=nst * 2 * b * n * es / ms / 1e6)
                    results.append(r)
                    print(json.dumps(r), flush=True)
                    if ok:
                        timings.append((ms, v))
                win = min(timings)[1] if timings else 0
                best[(logl, kind)] = win
                _lib.check(lib.tfft_tune_pass_select(pc, logl, kind, win))
        for (logl, kind), v in best.items():
            choice.setdefault(prec, {}).setdefault(logl, [0, 0, 0])[kind] = v
        del x, y
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(results, open(args.out, "w"), indent=1)
    print("PASS_CHOICE", json.dumps({p: {l: tuple(v) for l, v in sorted(d.items())}
                                     for p, d in choice.items()}))


if __name__ == "__main__":
    main()
