"""PCIe copy ceiling of the e2e number: pinned H2D, D2H and both at once
(separate streams), 1 GiB each, CUDA events."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "both"):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if name in ("h2d", "both"):
                s1.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if name in ("d2h", "both"):
                s2.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[name + "_GBps"] = round(n / best / 1e6, 1) * (2 if name == "both" else 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()


def host_path(logn=10, reps=5):
    """run_protected on a pinned 1 GiB host batch (the e2e path) vs the copy
    ceiling; prints ms per call."""
    import time
    import numpy as np
    from paper_2405_02520_b200 import Scheme, build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig
    from paper_2405_02520_b200.fft_core import fit_group_size
    n = 1 << logn
    b = (1 << 30) // (8 * n)
    xh = torch.randn(b, n, dtype=torch.complex64).pin_memory()
    plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
    tw = build_twiddles(plan)
    cfg = DetectionConfig(1e-4)
    run_protected(plan, tw, xh, Scheme.TWO_SIDED_GROUP, cfg)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, rep, _ = run_protected(plan, tw, xh, Scheme.TWO_SIDED_GROUP, cfg)
        ts.append((time.perf_counter() - t0) * 1e3)
        del out
    return {"logn": logn, "ms_host_path": round(min(ts), 2), "ms_median": round(sorted(ts)[len(ts) // 2], 2)}


if __name__ == "__main__" and len(__import__("sys").argv) > 1:
    import os
    print(json.dumps(host_path(int(__import__("sys").argv[1]))), os.environ.get("TFFT_STREAM_CHUNK_MB"))
