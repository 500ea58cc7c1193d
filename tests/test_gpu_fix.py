"""Device-side online correction (csrc/fix.cuh) of the single-kernel sizes:
the pass queued behind the fused launch (plan mode: it groups the flag
records itself) must give exactly the host-decided path's report and
outputs (tfft_set_device_correction(plan, 0): host decide() + the same
kernel in list mode), and the reference's decisions."""

import json

import numpy as np
import pytest
import torch

from conftest import random_batch

pytestmark = pytest.mark.gpu


def _plan(n, prec, b):
    from paper_2405_02520_b200 import make_plan
    from paper_2405_02520_b200.fft_core import fit_group_size
    return fit_group_size(make_plan(n, prec, batch=b), b)


def _run(plan, x, scheme, delta, inj_spec, device_fix):
    from paper_2405_02520_b200 import _lib, build_twiddles, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig
    from paper_2405_02520_b200.fault_lab import BitFlipInjector, FaultSpec
    from paper_2405_02520_b200.fft_core.plan import native_plan
    h = native_plan(plan, 0)
    lib = _lib.load()
    _lib.check(lib.tfft_set_device_correction(h.handle, int(device_fix)))
    try:
        inj = BitFlipInjector(FaultSpec(0, *inj_spec)) if inj_spec else None
        out, rep, cnt = run_protected(plan, build_twiddles(plan), torch.from_numpy(x).cuda(), scheme,
                                      DetectionConfig(delta), injector=inj)
        torch.cuda.synchronize()
        return out.cpu().numpy(), rep, cnt
    finally:
        _lib.check(lib.tfft_set_device_correction(h.handle, 1))


CASES = [  # (n, precision, batch)
    (8, "fp32", 128), (32, "fp32", 128), (1024, "fp32", 64), (2048, "fp32", 128), (8192, "fp32", 128),
    (64, "fp64", 128), (4096, "fp64", 128),
]


@pytest.mark.parametrize("n,prec,b", CASES)
@pytest.mark.parametrize("scheme", ["two_sided_group", "one_sided"])
def test_device_correction_equals_host_path_and_reference(n, prec, b, scheme):
    from oracle import port as P
    x = random_batch(np.random.default_rng([n, b]), (b, n), np.complex64 if prec == "fp32" else np.complex128)
    plan = _plan(n, prec, b)
    bs = plan.bs
    # several flags in one call: zero signals flag (0/0 -> inf, pipeline.py:118-121)
    # one in group 1, two in group 3 (unrecoverable when bs > 1), plus an
    # exponent flip of the output in group 5 (corrected)
    zeros = [1 * bs, 3 * bs + min(1, bs - 1) + (0 if bs > 1 else 1), 3 * bs]
    for z in zeros:
        x[z] = 0
    fault = (5 * bs + (bs - 1) // 2, n // 3, "im", 30 if prec == "fp32" else 62, "output")
    delta = 1e-4 if prec == "fp32" else 1e-9
    y_dev, rep_dev, cnt_dev = _run(plan, x, scheme, delta, fault, True)
    y_host, rep_host, cnt_host = _run(plan, x, scheme, delta, fault, False)
    assert rep_dev.to_json() == rep_host.to_json()
    assert rep_dev.max_rel_discrepancy == rep_host.max_rel_discrepancy
    assert cnt_dev.total == cnt_host.total
    np.testing.assert_array_equal(y_dev, y_host)
    # the reference's decisions on the same batch and fault
    op = P.shrink_bs(P.plan_for(n, prec, batch=b), b)
    _, orep, ocnt = P.protected(op, P.twiddles_for(op), x, scheme, delta=delta,
                                injector=P.OneShot(fault[0], fault[1], fault[2], fault[3]))
    mine = json.loads(rep_dev.to_json())
    for k in ("corrected", "unrecoverable", "recompute_count", "pass_count"):
        assert mine[k] == orep[k], (k, mine[k], orep[k])
    assert [(f["group"], f["signal"]) for f in mine["flagged"]] == \
           [(f["group"], f["signal"]) for f in orep["flagged"]]
    assert cnt_dev.total == ocnt.total
    assert fault[0] in [c["signal"] for c in mine["corrected"]]


def test_device_correction_many_jobs_one_sided():
    """delta far below the fp32 rounding noise: (almost) every signal flags;
    at bs = 1 (N = 1024) each is its own group, so the device pass plans and
    runs dozens of recompute jobs in one launch, exactly like the host path
    (and past 64 flags it hands the call to the host)."""
    n = 1024
    for b in (48, 96):
        x = random_batch(np.random.default_rng(b), (b, n), np.complex64)
        plan = _plan(n, "fp32", b)
        assert plan.bs == 1
        y_dev, rep_dev, _ = _run(plan, x, "one_sided", 1e-9, None, True)
        y_host, rep_host, _ = _run(plan, x, "one_sided", 1e-9, None, False)
        assert rep_dev.to_json() == rep_host.to_json()
        np.testing.assert_array_equal(y_dev, y_host)
        assert rep_dev.recompute_count == len(rep_dev.flagged) > 40
