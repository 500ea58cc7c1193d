"""Time N = 2048 / 4096 fp32 (ABFT on and off) with each ablation library
(tools/ablate_build.sh); prints one JSON line per (lib, n)."""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(logn, prec="fp32"):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2405_02520_b200 import _lib, make_plan
    from paper_2405_02520_b200.abft import make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan
    lib = _lib.load()
    for spec in filter(None, os.environ.get("TFFT_VARIANTS", "").split(",")):
        ln, var = (int(v) for v in spec.split(":"))
        if ln == logn:
            _lib.check(lib.tfft_tune_select(0, ln, var))
    n = 1 << logn
    dt, es = (torch.complex64, 8) if prec == "fp32" else (torch.complex128, 16)
    b = (1 << 30) // (es * n)
    x = torch.randn(b * n, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    plan = fit_group_size(make_plan(n, prec, batch=b), b)
    h = native_plan(plan, 0)
    row = make_encoding("wang", n).device_row(dt)
    rep = _lib.Report()
    sp = torch.cuda.current_stream().cuda_stream
    out = {}
    for sc in ("two_sided_group", "none"):
        code = _lib.SCHEME_CODE[sc]
        ts = []
        for i in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.tfft_run_protected(h.handle, x.data_ptr(), y.data_ptr(), b, code, 1e30, 0.0,
                                              row.data_ptr(), None, None, 0, ctypes.byref(rep), sp))
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        out[sc] = round(sorted(ts)[len(ts) // 2], 4)
    print(json.dumps({"lib": os.path.basename(os.environ.get("TFFT_LIB_PATH", "product")),
                      "variants": os.environ.get("TFFT_VARIANTS", ""), "prec": prec, "n": n, **out}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child(int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "fp32")
    else:
        libs = [None] + sorted(os.path.join(ROOT, "paper_2405_02520_b200", "ablate", f)
                               for f in os.listdir(os.path.join(ROOT, "paper_2405_02520_b200", "ablate")))
        for variants in ("",):
            for lib in libs:
                env = dict(os.environ)
                env["TFFT_VARIANTS"] = variants
                if lib:
                    env["TFFT_LIB_PATH"] = lib
                for spec in os.environ.get("ABLATE_SIZES", "fp32:11,fp32:12,fp32:13").split(","):
                    prec, logn = spec.split(":")
                    subprocess.run([sys.executable, __file__, "child", logn, prec], env=env)
