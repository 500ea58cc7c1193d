"""Minimal driver for ncu: a few protected (two_sided_group) launches of one
size on a 1 GiB batch, through the C ABI. Profile with e.g.

    ncu --set full --import-source on -k regex:fft_ -s 2 -c 1 -o prof \
        python tools/profile_single.py --prec fp32 --logn 12
"""

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="fp32")
    ap.add_argument("--logn", type=int, default=12)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--scheme", default="two_sided_group")
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--gib", type=float, default=1.0)
    a = ap.parse_args()
    import torch

    from paper_2405_02520_b200 import _lib, make_plan
    from paper_2405_02520_b200.abft import make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan

    lib = _lib.load()
    dt = torch.complex64 if a.prec == "fp32" else torch.complex128
    es = 8 if a.prec == "fp32" else 16
    n = 1 << a.logn
    total = int(a.gib * (1 << 30)) // es
    b = total // n
    x = torch.randn(b * n, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    plan = fit_group_size(make_plan(n, a.prec, batch=b), b)
    h = native_plan(plan, 0)
    row = make_encoding("wang", n).device_row(dt)
    pc = _lib.FP32 if a.prec == "fp32" else _lib.FP64
    if a.variant >= 0 and n <= 8192:
        _lib.check(lib.tfft_tune_select(pc, a.logn, a.variant))
    rep = _lib.Report()
    sp = torch.cuda.current_stream().cuda_stream
    code = _lib.SCHEME_CODE[a.scheme]
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off: skip setup kernels
    for _ in range(a.reps):
        _lib.check(lib.tfft_run_protected(h.handle, x.data_ptr(), y.data_ptr(), b, code,
                                          1e-4 if a.prec == "fp32" else 1e-9, 0.0,
                                          row.data_ptr(), None, None, 0, ctypes.byref(rep), sp))
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("done", a.prec, n, b, rep.n_flagged)


if __name__ == "__main__":
    main()
