"""BASELINE config C1 (the reference's own CPU-runnable case): batched FP32
N = 1024, batch 256, two-sided ABFT, no faults. A 4 MiB latency case (fits
L2): per-call wall time of run_protected through the public API (device
tensors; numpy in / out), and the fused launch alone (CUDA events), median
of 200 calls. Prints one JSON line."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import ctypes
    import numpy as np
    import torch
    from paper_2405_02520_b200 import Scheme, _lib, build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig, make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan
    n, b = 1024, 256
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(np.complex64)
    plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
    tw = build_twiddles(plan)
    cfg = DetectionConfig(1e-4)
    xd = torch.from_numpy(x).cuda()
    res = {"config": "C1: fp32 N=1024 batch=256 two_sided_group, no faults", "bs": plan.bs}
    for name, inp in (("device_api_us", xd), ("numpy_api_us", x)):
        for _ in range(20):
            run_protected(plan, tw, inp, Scheme.TWO_SIDED_GROUP, cfg)
        ts = []
        for _ in range(200):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run_protected(plan, tw, inp, Scheme.TWO_SIDED_GROUP, cfg)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e6)
        res[name] = round(statistics.median(ts), 1)
    lib = _lib.load()
    h = native_plan(plan, 0)
    row = make_encoding("wang", n).device_row(torch.complex64)
    y = torch.empty_like(xd)
    rep = _lib.Report()
    sp = torch.cuda.current_stream().cuda_stream
    ts = []
    for i in range(220):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.tfft_protect_launch(h.handle, xd.data_ptr(), y.data_ptr(), b, 3, 1e-4, 0.0,
                                           row.data_ptr(), None, None, 0, ctypes.byref(rep), sp))
        e1.record()
        torch.cuda.synchronize()
        _lib.check(lib.tfft_protect_finish(h.handle, xd.data_ptr(), y.data_ptr(), b, 3, 1e-4, 0.0,
                                           row.data_ptr(), None, 0, ctypes.byref(rep), sp))
        if i >= 20:
            ts.append(e0.elapsed_time(e1) * 1e3)
    res["fused_launch_us"] = round(statistics.median(ts), 1)
    res["gflops_device_api"] = round(5 * n * 10 * b / (res["device_api_us"] * 1e-6) / 1e9, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
