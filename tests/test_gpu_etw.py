"""The closed-form e^T W of the multi-pass first pass (multi.cuh
wang_cot_row: exactly reduced cot per thread + addition formula + Laurent
series near the pole, nothing read from memory) against the n-element table
it replaces (reference abft/encoding.py:58-62, pipeline.py:72-85).

The table path is the same fused kernel with ABFT_TABLE: passing the Wang
weights explicitly as a table encoding makes the first pass read the e^T W
row from memory. Decisions under identical injected faults must be equal,
flagged discrepancies within 1e-3, and the clean-data discrepancies of both
must be of the same (rounding-noise) size."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

# first-pass L >= 256 with batch <= 8 runs the closed form (multi_host.cu); the
# others the table in both arms (still a check of the dispatch)
CASES = [("fp32", 14, 64), ("fp32", 16, 8), ("fp32", 17, 4), ("fp32", 20, 8), ("fp64", 15, 32),
         ("fp64", 16, 8), ("fp64", 18, 4), ("fp64", 21, 4)]


def _run(lib, h, x, y, b, delta, row, vals, fault, inverse):
    from paper_2405_02520_b200 import _lib
    rep = _lib.Report()
    keep = ((_lib.Flag * 64)(), (ctypes.c_int64 * 64)(), (ctypes.c_int64 * 64)(), (ctypes.c_int64 * 64)())
    rep.flagged, rep.flagged_cap = keep[0], 64
    rep.corrected_group, rep.corrected_signal, rep.corrected_cap = keep[1], keep[2], 64
    rep.unrecoverable, rep.unrecoverable_cap = keep[3], 64
    _lib.check(lib.tfft_run_protected(h.handle, x.data_ptr(), y.data_ptr(), b, _lib.SCHEME_CODE["two_sided_group"],
                                      delta, 0.0, row.data_ptr(), vals.data_ptr() if vals is not None else None,
                                      ctypes.byref(fault) if fault is not None else None, int(inverse),
                                      ctypes.byref(rep), torch.cuda.current_stream().cuda_stream), "run")
    torch.cuda.synchronize()
    flags = sorted((int(keep[0][i].signal), float(keep[0][i].discrepancy)) for i in range(rep.n_flagged))
    corr = sorted(int(keep[2][i]) for i in range(rep.n_corrected))
    return flags, corr, int(rep.n_unrecoverable), float(rep.max_rel_discrepancy), y.clone()


@pytest.mark.parametrize("prec,logn,b", CASES)
@pytest.mark.parametrize("inverse", [False, True])
def test_closed_form_row_matches_table(prec, logn, b, inverse):
    from paper_2405_02520_b200 import _lib, make_plan
    from paper_2405_02520_b200.abft import make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan
    lib = _lib.load()
    n = 1 << logn
    td = torch.complex64 if prec == "fp32" else torch.complex128
    plan = fit_group_size(make_plan(n, prec, batch=b), b)
    h = native_plan(plan, 0)
    enc = make_encoding("wang", n)
    row = enc.device_row(td, inverse)
    vals = enc.values_dev.to(td).contiguous()  # Wang weights as an explicit table: ABFT_TABLE path
    g = torch.Generator(device="cuda").manual_seed(logn)
    x = torch.randn((b, n), dtype=td, device="cuda", generator=g)
    y = torch.empty_like(x)
    delta = 1e-4 if prec == "fp32" else 1e-9
    bit = 30 if prec == "fp32" else 62
    clean_cf = _run(lib, h, x, y, b, delta, row, None, None, inverse)
    clean_tb = _run(lib, h, x, y, b, delta, row, vals, None, inverse)
    assert clean_cf[0] == clean_tb[0] == []
    assert torch.equal(clean_cf[4], clean_tb[4])  # the checksums never touch the outputs
    # the clean max discrepancy is rounding noise in both: same order of magnitude
    assert clean_cf[3] < 10 * clean_tb[3] + (1e-7 if prec == "fp32" else 1e-15)
    rng = np.random.default_rng(logn + 7)
    for where in (_lib.AT_INPUT, _lib.AT_OUTPUT):
        f = _lib.Fault()
        f.signal, f.element = int(rng.integers(b)), int(rng.integers(n))
        f.component, f.bit, f.where = int(rng.integers(2)), bit, where
        cf = _run(lib, h, x, y, b, delta, row, None, f, inverse)
        tb = _run(lib, h, x, y, b, delta, row, vals, f, inverse)
        assert [s for s, _ in cf[0]] == [s for s, _ in tb[0]], (where, cf[0], tb[0])
        if where == _lib.AT_INPUT:  # |x| < 2: the exponent flip makes it ~1e38 -> always flagged
            assert [s for s, _ in cf[0]] == [f.signal]
        # (an output flip of a component with 2 <= |y| < ~delta |c_in| is sub-threshold
        # in both: decisions must agree, detection is not guaranteed)
        assert cf[1] == tb[1] and cf[2] == tb[2]
        for (_, a), (_, c) in zip(cf[0], tb[0]):
            assert a == pytest.approx(c, rel=1e-3) or (np.isinf(a) and np.isinf(c))
