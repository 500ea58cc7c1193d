"""Host-side profile of the C1 call (FP32 N = 1024, batch 256, device
tensors): cProfile of 300 public run_protected calls, top functions by
internal time. Shows where the ~40 us of host work per call goes."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2405_02520_b200 import Scheme, build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig
    from paper_2405_02520_b200.fft_core import fit_group_size
    n, b = 1024, 256
    x = np.random.default_rng(0).standard_normal((b, 2 * n)).view(np.complex128).astype(np.complex64)
    plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
    tw = build_twiddles(plan)
    cfg = DetectionConfig(1e-4)
    xd = torch.from_numpy(x).cuda()
    for _ in range(50):
        run_protected(plan, tw, xd, Scheme.TWO_SIDED_GROUP, cfg)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(300):
        run_protected(plan, tw, xd, Scheme.TWO_SIDED_GROUP, cfg)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
