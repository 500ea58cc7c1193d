"""Parity at the benchmark's own scale (bench.py C2 / C3 batches).

* Every C2 size (fp32 N = 2^3..2^13, 1 GiB batch) and C3 size (fp64
  N = 2^20..2^25, 2 GiB batch): the protected output equals the unprotected
  output bitwise (the reference's fusion contract, test_abft.py:265-273), and
  >= 64 sampled signals (first / last, tile and grid-stride boundaries,
  random) match an fp64 FFT within 2e-7 (fp32) / 1e-15 (fp64) x log2 n
  per-signal relative L2.
* Clean-data flags of the full C2 sweep. A clean signal is flagged when the
  rounding noise of c_in - c_out (fp32 sums and fp32 FFT, here and in the
  reference alike) exceeds delta * |c_in|, i.e. only for signals whose
  |c_in| is tiny. The noise of two implementations that round in different
  orders is correlated but not equal, so a signal picked for being the
  largest of ~10^7 draws of OUR noise is typically smaller in the
  reference's draw (selection effect; an fp32 emulation of this kernel's
  summation order vs the reference on 2^20 signals at N = 64 gives 19 / 22
  signals above 3e-5 but the top signals differ by up to 6x). So:
  - every full-scale clean flag must lie in the reference's own far noise
    tail: its reference rel > delta / 30 (a median clean rel is ~1e-7 to
    5e-7, i.e. this is the top ~0.1 % of the reference's distribution);
  - our noise must not exceed the reference's: on a common random sample per
    size, the number of signals above a probe threshold (1e-6 .. 3e-6, ~10^3
    signals in the reference) is at most 1.5x the reference's (measured: at
    N = 1024 ours is ~3x lower);
  - on a 2^18-sample of every size the decisions at delta agree wherever the
    reference's discrepancy is outside [delta / 10, 10 delta].
  TFFT_SCALE_DUMP=path writes the summary as JSON.
"""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

C2 = list(range(3, 14))
C3 = list(range(20, 26))


def _plan(n, prec, b):
    from paper_2405_02520_b200 import make_plan
    from paper_2405_02520_b200.fft_core import fit_group_size
    return fit_group_size(make_plan(n, prec, batch=b), b)


def _sample_idx(b, rng, k=64):
    idx = {0, 1, 2, 3, b - 1, b - 2, b - 3}
    for j in range(1, 24):
        for e in (148 * j, 148 * 2 * j, 1 << j):  # grid-stride / power-of-two tile boundaries
            for d in (-1, 0):
                if 0 <= e + d < b:
                    idx.add(e + d)
    idx.update(rng.choice(b, size=min(b, k), replace=False).tolist())
    return np.array(sorted(i for i in idx if 0 <= i < b))


def _run(plan, x, scheme, delta):
    from paper_2405_02520_b200 import build_twiddles, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig
    return run_protected(plan, build_twiddles(plan), x, scheme, DetectionConfig(delta))


def _check_size(prec, logn, total_bytes, seed, summary):
    n = 1 << logn
    esz = 8 if prec == "fp32" else 16
    td = torch.complex64 if prec == "fp32" else torch.complex128
    b = total_bytes // (n * esz)
    plan = _plan(n, prec, b)
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((b, n), dtype=td, device="cuda", generator=g)
    delta = 1e-4 if prec == "fp32" else 1e-9
    y_on, rep, _ = _run(plan, x, "two_sided_group", delta)
    y_off, _, _ = _run(plan, x, "none", delta)
    # fusion contract: bitwise equal except the signals a (clean-data) flag
    # got corrected: those were rebuilt as W s0 - sum of the others and
    # re-verified (pipeline.py:180-191), equal to the FFT only to rounding
    fixed = sorted({c["signal"] for c in rep.corrected})
    rv = torch.float32 if prec == "fp32" else torch.float64
    keep = torch.ones(b, dtype=torch.bool, device="cuda")
    if fixed:
        keep[torch.tensor(fixed, device="cuda")] = False
    assert torch.equal(y_on[keep].view(rv), y_off[keep].view(rv)), (prec, n)
    del y_off
    idx = np.union1d(_sample_idx(b, np.random.default_rng([seed, logn])), np.array(fixed, dtype=np.int64))
    it = torch.from_numpy(idx).cuda()
    xs = x.index_select(0, it).cpu().numpy().astype(np.complex128)
    ys = y_on.index_select(0, it).cpu().numpy().astype(np.complex128)
    ref = np.fft.fft(xs, axis=1)
    err = np.linalg.norm(ys - ref, axis=1) / np.linalg.norm(ref, axis=1)
    tol = (2e-7 if prec == "fp32" else 1e-15) * logn
    assert err.max() <= tol, (prec, n, float(err.max()), int(idx[err.argmax()]))
    summary.setdefault("sizes", []).append(
        {"prec": prec, "n": n, "batch": b, "sampled": len(idx), "max_rel_l2": float(err.max()),
         "flagged": len(rep.flagged), "unrecoverable": len(rep.unrecoverable),
         "corrected": len(rep.corrected)})
    flagged = [(f["signal"], f["discrepancy"]) for f in rep.flagged]
    xh = None
    if flagged:
        sig = torch.tensor(sorted({s for s, _ in flagged}), device="cuda")
        xh = {int(s): v for s, v in zip(sig.tolist(), x.index_select(0, sig).cpu().numpy())}
    del x, y_on
    torch.cuda.empty_cache()
    return plan, flagged, xh


def test_c3_fp64_bench_scale():
    summary = {}
    for logn in C3:
        _check_size("fp64", logn, 2 << 30, 4321, summary)
    for s in summary["sizes"]:
        assert s["flagged"] == 0, s  # fp64 clean data: no false alarms at delta 1e-9


def _ref_rel(row, kernel):
    """The reference's rel of one signal: its row through the reference's
    encode / transform / verify as a group of one (c_in, c_out and the floor
    are per-signal quantities, pipeline.py:72-135)."""
    from oracle import port as P
    n = row.shape[-1]
    xg = np.asarray(row, dtype=np.complex64)[None, :]
    enc = P.encoding_for("wang", n, kernel)
    p1 = P.shrink_bs(P.plan_for(n, "fp32", batch=1), 1)
    st = P.encode(xg, enc)
    yg = P.execute(p1, P.twiddles_for(p1), xg.copy(), kernel=kernel)
    _, rr, _ = P.verify(st, yg, enc, 1e-4, 0.0, "fp32")
    return float(rr[0])


def test_c2_fp32_bench_scale_and_clean_flags_vs_reference():
    from oracle import port as P
    kernel = "ref" if P.have_ref_kernel() else "c"
    summary = {"kernel": kernel}
    flags = []
    for logn in C2:
        plan, flagged, xh = _check_size("fp32", logn, 1 << 30, 1234, summary)
        n = 1 << logn
        for s, rel in flagged:
            flags.append({"n": n, "signal": int(s), "rel_ours": float(rel),
                          "rel_reference": _ref_rel(xh[s], kernel)})
    summary["clean_flags"] = flags
    for f in flags:
        assert f["rel_reference"] > 1e-4 / 30, f  # outside the reference's own noise tail: fail
    summary["flags_reference_also_flags"] = sum(f["rel_reference"] > 1e-4 for f in flags)
    # random sample of every size: decisions agree outside the x3 band
    rng = np.random.default_rng(99)
    sample = []
    for logn in C2:
        n = 1 << logn
        b = max(16, (1 << 18) // n) // 16 * 16
        x = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(np.complex64)
        plan = _plan(n, "fp32", b)
        _, rep, _ = _run(plan, torch.from_numpy(x).cuda(), "two_sided_group", 1e-4)
        mine = {f["signal"] for f in rep.flagged}
        op = P.shrink_bs(P.plan_for(n, "fp32", batch=b), plan.bs)
        _, orep, _ = P.protected(op, P.twiddles_for(op), x, "two_sided_group", delta=1e-4,
                                 enc=P.encoding_for("wang", n, kernel), kernel=kernel)
        theirs = {f["signal"]: f["discrepancy"] for f in orep["flagged"]}
        for s in mine ^ set(theirs):
            r = theirs[s] if s in theirs else _ref_rel(x[s], kernel)
            assert 1e-4 / 10 < r < 1e-3, (n, s, r)
        sample.append({"n": n, "signals": b, "ours_flagged": len(mine), "reference_flagged": len(theirs)})
    summary["random_sample"] = sample
    summary["noise_tail"] = _noise_tails(kernel)
    dump = os.environ.get("TFFT_SCALE_DUMP")
    if dump:
        with open(dump, "w") as f:
            json.dump(summary, f, indent=1)


def _noise_tails(kernel):
    """Counts of clean signals whose rel exceeds a probe threshold, ours (the
    fused kernel's flag records at delta = probe) vs the reference's, on the
    same seeded sample; ~10^3 signals each, so binomial noise is ~3 %."""
    from oracle import port as P
    out = []
    for n, b, probe in ((8, 1 << 21, 3e-6), (64, 1 << 20, 3e-6), (1024, 1 << 16, 3e-6), (8192, 1 << 13, 1e-6)):
        rng = np.random.default_rng([7, n])
        x = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(np.complex64)
        plan = _plan(n, "fp32", b)
        _, rep, _ = _run(plan, torch.from_numpy(x).cuda(), "two_sided_group", probe)
        ours = {f["signal"] for f in rep.flagged}
        enc = P.encoding_for("wang", n, kernel)
        p1 = P.shrink_bs(P.plan_for(n, "fp32", batch=1), 1)
        tw = P.twiddles_for(p1)
        y = np.concatenate([P.execute(p1, tw, x[i:i + 1024].copy(), kernel=kernel) for i in range(0, b, 1024)])
        _, rr, _ = P.verify(P.encode(x, enc), y, enc, probe, 0.0, "fp32")
        theirs = set(np.flatnonzero(rr > probe).tolist())
        rec = {"n": n, "signals": b, "probe": probe, "ours": len(ours), "reference": len(theirs),
               "both": len(ours & theirs)}
        out.append(rec)
        assert len(theirs) >= 100, rec
        assert len(ours) <= 1.5 * len(theirs), rec  # no noisier than the reference
    return out
