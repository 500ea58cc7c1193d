"""e2e (host-buffer) throughput of the C2 sweep through the public
run_protected for one streaming chunk size (TFFT_STREAM_CHUNK_MB is read once
per process, so run one process per size), next to the PCIe copy ceiling.

    for mb in 16 32 64 128; do TFFT_STREAM_CHUNK_MB=$mb python tools/e2e_chunks.py; done
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2405_02520_b200 import Scheme, build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig
    from paper_2405_02520_b200.fft_core import fit_group_size
    xh = torch.randn((1 << 30) // 8, dtype=torch.complex64).pin_memory()
    cfg = DetectionConfig(1e-4)
    cases = []
    for logn in range(3, 14):
        n = 1 << logn
        b = (1 << 30) // (8 * n)
        plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
        cases.append((plan, build_twiddles(plan), xh[:b * n].view(b, n)))

    def step():
        for plan, tw, xv in cases:
            run_protected(plan, tw, xv, Scheme.TWO_SIDED_GROUP, cfg)
    step()
    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1000 / reps
    fl = sum(5.0 * p.n * math.log2(p.n) * xv.shape[0] for p, _, xv in cases)
    print(json.dumps({"chunk_mb": os.environ.get("TFFT_STREAM_CHUNK_MB", "32 (default)"), "ms_per_step": round(ms, 2),
                      "gflops": round(fl / (ms / 1000) / 1e9, 1)}))


if __name__ == "__main__":
    main()
