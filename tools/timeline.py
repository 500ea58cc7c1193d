"""Device timeline of one protected call (torch.profiler / CUPTI): every
kernel, memcpy and memset with its start offset and duration, for a clean
call and for a call with one injected fault, so the online-correction cost
can be attributed (there is no nsys in this image).

    python tools/timeline.py --prec fp32 --logn 16 [--gib 1] [--bit 30]
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="fp32")
    ap.add_argument("--logn", type=int, default=16)
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--bit", type=int, default=None)
    ap.add_argument("--where", default="output")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2405_02520_b200 import Scheme, build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig
    from paper_2405_02520_b200.fault_lab import BitFlipInjector, FaultSpec
    from paper_2405_02520_b200.fft_core import fit_group_size

    n = 1 << a.logn
    dt = torch.complex64 if a.prec == "fp32" else torch.complex128
    esz = 8 if a.prec == "fp32" else 16
    b = int(a.gib * (1 << 30)) // (esz * n)
    bit = a.bit if a.bit is not None else (30 if a.prec == "fp32" else 62)
    x = torch.randn((b, n), dtype=dt, device="cuda")
    plan = fit_group_size(make_plan(n, a.prec, batch=b), b)
    tw = build_twiddles(plan)
    cfg = DetectionConfig(1e-4 if a.prec == "fp32" else 1e-9)

    def call(fault):
        inj = BitFlipInjector(FaultSpec(0, b // 2 + 3, n // 3, "re", bit, a.where)) if fault else None
        out, rep, _ = run_protected(plan, tw, x, Scheme.TWO_SIDED_GROUP, cfg, injector=inj)
        return rep

    for _ in range(3):
        call(False), call(True)
    torch.cuda.synchronize()
    for fault in (False, True):
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            rep = call(fault)
            torch.cuda.synchronize()
        evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
        evs.sort(key=lambda e: e.time_range.start)
        t0 = evs[0].time_range.start if evs else 0
        print(f"== {'one fault' if fault else 'clean'}: n={n} batch={b} flagged={len(rep.flagged)} "
              f"corrected={len(rep.corrected)}")
        last = t0
        for e in evs:
            st, en = e.time_range.start, e.time_range.end
            print(f"  +{(st - t0):9.1f} us  gap {(st - last):7.1f}  dur {(en - st):8.1f}  {e.name[:100]}")
            last = max(last, en)
        cpu = [e for e in prof.events() if e.device_type.name == "CPU" and e.name.startswith(("cuda", "aten"))]
        tot = sum(e.time_range.end - e.time_range.start for e in cpu)
        print(f"  device span {(last - t0):.1f} us; CPU-side cuda*/aten* calls {len(cpu)} ({tot:.1f} us)")


if __name__ == "__main__":
    main()
