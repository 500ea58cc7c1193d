"""GPU ABFT parity: detection / correction decisions under identical injected
faults must equal the reference's (bit-exact decisions), outputs within the
stated tolerance, and the reference's fusion / pass-count contracts hold."""

import json
import math
import os

import numpy as np
import pytest
import torch

from conftest import ROOT, random_batch, rel_l2
from golden.make_golden import protected_input

pytestmark = pytest.mark.gpu

from paper_2405_02520_b200.abft import (DetectionConfig, Scheme, UnrecoverableError,  # noqa: E402
                                        correct_group, detect, encode_group, finalize_group,
                                        make_encoding, run_protected)
from paper_2405_02520_b200.fault_lab import BitFlipInjector, FaultSpec  # noqa: E402
from paper_2405_02520_b200.fft_core import (build_twiddles, fft_execute, fit_group_size,  # noqa: E402
                                            make_plan)

GOLD = os.path.join(ROOT, "tests", "golden")
TOL = {"fp32": 1e-5, "fp64": 1e-12}


def decisions(rep):
    d = rep if isinstance(rep, dict) else json.loads(rep.to_json())
    return ([(f["group"], f["signal"]) for f in d["flagged"]],
            [(c["group"], c["signal"]) for c in d["corrected"]],
            list(d["unrecoverable"]), d["recompute_count"], d["pass_count"])


def test_golden_protected_cases():
    from oracle import port as P
    cases = json.load(open(os.path.join(GOLD, "protected.json")))
    arrays = np.load(os.path.join(GOLD, "protected.npz"))
    for c in cases:
        x = protected_input(c["id"], c["n"], c["batch"], c["precision"])
        plan = fit_group_size(make_plan(c["n"], c["precision"], batch=c["batch"]), c["batch"])
        inj = None
        if c["fault"] is not None:
            s, el, comp, bit, stage = c["fault"]
            inj = BitFlipInjector(FaultSpec(0, s, el, comp, bit, stage))
        cfg = DetectionConfig(delta=1e-4 if c["precision"] == "fp32" else 1e-9)
        out, rep, cnt = run_protected(plan, build_twiddles(plan), torch.from_numpy(x).cuda(),
                                      c["scheme"], cfg, injector=inj, inverse=c["inverse"])
        assert decisions(rep) == decisions(c["report"]), c["id"]
        assert cnt.total == c["pass_total"]
        assert (inj.fired if inj else False) == c["fired"]
        for mine, theirs in zip(rep.flagged, c["report"]["flagged"]):
            if math.isinf(theirs["discrepancy"]):
                assert math.isinf(mine["discrepancy"])
            else:
                assert mine["discrepancy"] == pytest.approx(theirs["discrepancy"], rel=1e-3)
        key = f"c{c['id']}_y"
        if key in arrays:
            ref = arrays[key]
        else:  # oracle (pinned bit-exact to the reference by test_oracle.py)
            op = P.shrink_bs(P.plan_for(c["n"], c["precision"], batch=c["batch"]), c["batch"])
            oinj = P.OneShot(*c["fault"]) if c["fault"] else None
            ref, _, _ = P.protected(op, P.twiddles_for(op), x, c["scheme"],
                                    delta=cfg.delta, injector=oinj, inverse=c["inverse"])
        tol = TOL[c["precision"]] * math.log2(c["n"]) * (10 if c["report"]["corrected"] else 1)
        assert rel_l2(out, ref) <= tol, (c["id"], rel_l2(out, ref))


@pytest.mark.parametrize("n,prec", [(16, "fp32"), (256, "fp32"), (1024, "fp32"), (8192, "fp64"),
                                    (2**14, "fp64"), (2**17, "fp32"), (2**23, "fp32")])
def test_fusion_bitwise_and_pass_count(n, prec):
    b = 16 if n <= 2**17 else 2
    x = random_batch(np.random.default_rng(5), (b, n), np.complex64 if prec == "fp32"
                     else np.complex128)
    plan = make_plan(n, prec, batch=b)
    plan = fit_group_size(plan, b)
    tw = build_twiddles(plan)
    xd = torch.from_numpy(x).cuda()
    cfg = DetectionConfig(delta=1e-4 if prec == "fp32" else 1e-9)
    clean, _, c0 = run_protected(plan, tw, xd, Scheme.NONE, cfg)
    prot, rep, c2 = run_protected(plan, tw, xd, Scheme.TWO_SIDED_GROUP, cfg)
    assert torch.equal(clean, prot)
    assert c0.total == c2.total == 2 * len(plan.stages) * (b // plan.bs)
    assert rep.flagged == [] and rep.recompute_count == 0
    assert 0 < rep.max_rel_discrepancy < cfg.delta
    assert torch.equal(clean, fft_execute(plan, tw, xd))


def test_exponent_bit_flips_all_detected_and_corrected():
    """Reference acceptance 04 (tests/test_acceptance.py:104-141), with every
    decision also compared against the oracle."""
    from oracle import port as P
    plan = make_plan(256, "fp32", batch=8)
    tw = build_twiddles(plan)
    op = P.plan_for(256, "fp32", batch=8)
    otw = P.twiddles_for(op)
    cfg = DetectionConfig(delta=1e-4)
    detected = corrected = rec_two = rec_one = 0
    total = 200
    for i in range(total):
        rng = np.random.default_rng([77, i])
        x = random_batch(rng, (8, 256), np.complex64)
        spec = FaultSpec(i, int(rng.integers(8)), int(rng.integers(256)),
                         "re" if rng.integers(2) == 0 else "im", int(rng.integers(25, 31)))
        xd = torch.from_numpy(x).cuda()
        clean, _, _ = run_protected(plan, tw, xd, Scheme.NONE, cfg)
        out, rep, _ = run_protected(plan, tw, xd, Scheme.TWO_SIDED_GROUP, cfg,
                                    injector=BitFlipInjector(spec))
        _, orep, _ = P.protected(op, otw, x, "two_sided_group", delta=1e-4,
                                 injector=P.OneShot(spec.signal_idx, spec.element_idx,
                                                    spec.component, spec.bit))
        assert decisions(rep) == decisions(orep)
        rec_two += rep.recompute_count
        if rep.flagged:
            detected += 1
            if rel_l2(out, clean) <= 1e-4:
                corrected += 1
        _, rep1, _ = run_protected(plan, tw, xd, Scheme.ONE_SIDED, cfg,
                                   injector=BitFlipInjector(spec))
        rec_one += rep1.recompute_count
    assert detected == total and corrected == detected
    assert rec_two == 0 and rec_one == detected


@pytest.mark.parametrize("n,prec,stage", [(2**14, "fp64", "stage:0"), (2**14, "fp32", "stage:1"),
                                          (2**23, "fp64", "stage:1"), (2**20, "fp64", "input"),
                                          (2**25, "fp32", "output"), (2**23, "fp32", "stage:2"),
                                          # 2-stage API plans executed as 3 passes (fast split) unless a
                                          # stage:k hook needs the API plan's intermediates
                                          (2**21, "fp64", "output"), (2**22, "fp64", "input"),
                                          (2**22, "fp32", "stage:0"), (2**21, "fp32", "stage:1")])
def test_multipass_injection_corrected(n, prec, stage):
    b = 2
    x = random_batch(np.random.default_rng(n), (b, n), np.complex64 if prec == "fp32"
                     else np.complex128)
    plan = fit_group_size(make_plan(n, prec, batch=b), b)
    tw = build_twiddles(plan)
    xd = torch.from_numpy(x).cuda()
    cfg = DetectionConfig(delta=1e-4 if prec == "fp32" else 1e-9)
    clean, _, _ = run_protected(plan, tw, xd, Scheme.NONE, cfg)
    # top exponent bit for inputs (|x| < 2: x 2^128 / 2^1024), the next one for
    # stage / output values (|v| >= 2 there: x 2^64 / 2^512) - a flip that
    # always grows the value, so the fault is never subthreshold
    bit = (30 if prec == "fp32" else 62) - (stage != "input")
    inj = BitFlipInjector(FaultSpec(0, 1, n // 3 + 7, "re", bit, stage))
    out, rep, _ = run_protected(plan, tw, xd, Scheme.TWO_SIDED_GROUP, cfg, injector=inj)
    assert inj.fired
    assert [c["signal"] for c in rep.corrected] == [1], rep.to_json()
    assert rel_l2(out, clean) <= TOL[prec] * math.log2(n) * 10


def test_double_fault_unrecoverable_generic_callable():
    plan = fit_group_size(make_plan(256, "fp64", batch=8), 8)
    x = random_batch(np.random.default_rng(1), (8, 256))

    def double_fault(where, group_start, buf):
        if where == "output":
            buf[0, 0] += 100.0
            buf[3, 9] += 100.0

    out, rep, _ = run_protected(plan, build_twiddles(plan), torch.from_numpy(x).cuda(),
                                Scheme.TWO_SIDED_GROUP, DetectionConfig(delta=1e-9),
                                injector=double_fault)
    assert rep.unrecoverable == [0] and rep.corrected == []


def test_generic_callable_matches_fused_path():
    plan = fit_group_size(make_plan(2**14, "fp64", batch=4), 4)
    tw = build_twiddles(plan)
    x = torch.from_numpy(random_batch(np.random.default_rng(2), (4, 2**14))).cuda()
    cfg = DetectionConfig(delta=1e-9)
    spec = FaultSpec(0, 2, 999, "re", 62, "stage:0")
    a, ra, ca = run_protected(plan, tw, x, Scheme.TWO_SIDED_GROUP, cfg,
                              injector=BitFlipInjector(spec))
    inj = BitFlipInjector(spec)
    b, rb, cb = run_protected(plan, tw, x, Scheme.TWO_SIDED_GROUP, cfg,
                              injector=lambda w, s, buf: inj(w, s, buf))
    assert decisions(ra) == decisions(rb) and ca.total == cb.total
    assert rel_l2(a, b) <= 1e-13


def test_pipeline_api_zero_batch_and_inf():
    plan = make_plan(8, "fp64")
    tw = build_twiddles(plan)
    enc = make_encoding("ones", 8)
    xg = torch.zeros(4, 8, dtype=torch.complex128, device="cuda")
    state = encode_group(xg, enc)
    yg = fft_execute(plan, tw, xg)
    yg[1, 2] += 1.0
    finalize_group(state, yg)
    fixed = correct_group(state, yg, 1, plan, tw, enc, DetectionConfig(delta=1e-4, abs_floor=1e-12))
    assert torch.equal(fixed, torch.zeros_like(fixed))
    rng = np.random.default_rng(0)
    x = torch.from_numpy(random_batch(rng, (4, 8))).cuda()
    st = encode_group(x, enc)
    y = fft_execute(plan, tw, x)
    y[1, 0] = float("inf")
    rep = detect(st, y, enc, DetectionConfig(delta=1e30))
    assert [f.signal_idx for f in rep.flagged] == [1]


def test_pipeline_api_unit_fault_and_corrupted_checksum():
    plan = make_plan(8, "fp64")
    tw = build_twiddles(plan)
    enc = make_encoding("ones", 8)
    x = torch.from_numpy(random_batch(np.random.default_rng(3), (4, 8))).cuda()
    clean = fft_execute(plan, tw, x)
    st = encode_group(x, enc)
    y = clean.clone()
    y[0, 0] += 1.0
    rep = detect(st, y, enc, DetectionConfig(delta=1e-4))
    assert [f.signal_idx for f in rep.flagged] == [0]
    assert abs(abs(rep.flagged[0].epsilon_estimate) - 1.0) < 1e-9
    y2 = clean.clone()
    y2[2, 5] += 1.0
    fixed = correct_group(st, y2, 2, plan, tw, enc, DetectionConfig(delta=1e-4))
    assert rel_l2(fixed, clean) <= 1e-10
    y3 = clean.clone()
    y3[0] += 1.0
    y3[3, 1] += 5.0
    with pytest.raises(UnrecoverableError):
        correct_group(st, y3, 3, plan, tw, enc, DetectionConfig(delta=1e-4))


def test_encodings_match_reference_golden():
    g = np.load(os.path.join(GOLD, "encodings.npz"))
    for kind in ("wang", "ones", "jou", "linear"):
        for n in (2, 4, 16, 1024):
            enc = make_encoding(kind, n)
            ref = g[f"{kind}_{n}_etw"]
            scale = max(np.abs(ref).max(), 1.0)
            assert np.abs(enc.etw - ref).max() <= 1e-12 * scale
            assert np.abs(enc.etw_inv - g[f"{kind}_{n}_etw_inv"]).max() <= 1e-12 * scale


def test_zero_signals_flag_without_floor():
    """rel = 0/0 -> NaN -> inf flags (reference pipeline.py:116-121)."""
    plan = fit_group_size(make_plan(64, "fp32", batch=4), 4)
    x = torch.zeros(4, 64, dtype=torch.complex64, device="cuda")
    _, rep, _ = run_protected(plan, build_twiddles(plan), x, Scheme.TWO_SIDED_GROUP)
    assert [f["signal"] for f in rep.flagged] == [0, 1, 2, 3]
    assert rep.unrecoverable == [0]
    _, rep2, _ = run_protected(plan, build_twiddles(plan), x, Scheme.TWO_SIDED_GROUP,
                               DetectionConfig(delta=1e-4, abs_floor=1e-12))
    assert rep2.flagged == []


@pytest.mark.parametrize("n,prec,batch", [(1024, "fp32", 10000), (1 << 16, "fp64", 48), (64, "fp32", 16)])
@pytest.mark.parametrize("scheme", ["two_sided_group", "one_sided", "none"])
def test_host_streaming_matches_device_path(n, prec, batch, scheme):
    """tfft_run_protected_host (numpy in -> numpy out, chunked H2D / transform /
    D2H on three streams) gives the device path's outputs bit for bit and the
    same report, with the fault landing in the last chunk."""
    dt = np.complex64 if prec == "fp32" else np.complex128
    x = random_batch(np.random.default_rng(7), (batch, n), dt)
    plan = fit_group_size(make_plan(n, prec, batch=batch), batch)
    tw = build_twiddles(plan)
    cfg = DetectionConfig(delta=1e-4 if prec == "fp32" else 1e-9)
    spec = FaultSpec(0, batch - 3, n // 3, "re", 30 if prec == "fp32" else 62)
    yd, rd, cd = run_protected(plan, tw, torch.from_numpy(x).cuda(), scheme, cfg,
                               injector=BitFlipInjector(spec))
    inj = BitFlipInjector(spec)
    yh, rh, ch = run_protected(plan, tw, x, scheme, cfg, injector=inj)
    assert isinstance(yh, np.ndarray) and yh.dtype == x.dtype
    assert np.array_equal(yh.view(np.uint8), yd.cpu().numpy().view(np.uint8))
    assert rh.to_json() == rd.to_json()
    assert ch.total == cd.total
    assert inj.fired
    if scheme != "none":
        assert [c["signal"] for c in rh.corrected] == [batch - 3]


@pytest.mark.parametrize("n,prec,device_input", [(1024, "fp32", True), (1 << 15, "fp64", True),
                                                 (256, "fp32", False)])
def test_floor_recheck_path_matches_oracle(n, prec, device_input):
    """Signals with c_in ~ 0 (orthogonal to e^T W) make the detection floor
    FLOOR_COEF * sum|x| decide; the kernels cannot settle that from their l1
    upper bound and send them to the exact recheck. Their flags and rel must
    be the reference's (oracle port), mixed with ordinary signals."""
    from oracle import port as P
    dt = np.complex64 if prec == "fp32" else np.complex128
    rng = np.random.default_rng(21)
    b = 8
    x = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n)))
    etw = P.encoding_for("wang", n).etw
    for s in (1, 2, 5):  # project out the checksum direction
        x[s] -= (x[s] @ etw) * np.conj(etw) / np.vdot(etw, etw).real
    x = x.astype(dt)
    plan = fit_group_size(make_plan(n, prec, batch=b), 1)
    delta = 1e-4 if prec == "fp32" else 1e-9
    xin = torch.from_numpy(x).cuda() if device_input else x
    _, rep, _ = run_protected(plan, build_twiddles(plan), xin, Scheme.TWO_SIDED_GROUP, DetectionConfig(delta))
    op = P.shrink_bs(P.plan_for(n, prec, batch=b), 1)
    _, orep, _ = P.protected(op, P.twiddles_for(op), x, "two_sided_group", delta=delta)
    assert [f["signal"] for f in rep.flagged] == [f["signal"] for f in orep["flagged"]]
    assert {1, 2, 5} <= {f["signal"] for f in rep.flagged}
    # c_in and c_out of these signals are rounding noise of two different FFT
    # implementations: the values agree in magnitude, far above delta
    for mine, theirs in zip(rep.flagged, orep["flagged"]):
        assert mine["discrepancy"] > 10 * delta and theirs["discrepancy"] > 10 * delta
        assert 0.2 < mine["discrepancy"] / theirs["discrepancy"] < 5
    assert rep.max_rel_discrepancy > 0 and math.isfinite(rep.max_rel_discrepancy)


def test_thread_level_check_level():
    """Check level 1 (the paper's thread-level scheme, scheme comparison
    only): outputs bitwise equal to the unprotected transform, no false
    alarms on clean data. It verifies each radix tile's DFT, so corruption of
    the data between tiles (an "input" fault here) is outside its coverage —
    while the default threadblock checksums catch and correct it."""
    from paper_2405_02520_b200 import _lib
    from paper_2405_02520_b200.fft_core.plan import native_plan
    n, b = 1024, 64
    x = random_batch(np.random.default_rng(4), (b, n), np.complex64)
    plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
    tw = build_twiddles(plan)
    ref, _, _ = run_protected(plan, tw, torch.from_numpy(x).cuda(), Scheme.NONE)
    h = native_plan(plan, torch.cuda.current_device())
    spec = FaultSpec(0, 9, 100, "re", 26, "input")  # finite (x 2^8): consistent inside every tile
    _lib.check(_lib.load().tfft_set_check_level(h.handle, 1))
    try:
        y, rep, _ = run_protected(plan, tw, torch.from_numpy(x).cuda(), Scheme.TWO_SIDED_GROUP)
        assert rep.flagged == [] and torch.equal(y, ref)
        _, rep, _ = run_protected(plan, tw, torch.from_numpy(x).cuda(), Scheme.TWO_SIDED_GROUP,
                                  injector=BitFlipInjector(spec))
        assert rep.flagged == []
    finally:
        _lib.check(_lib.load().tfft_set_check_level(h.handle, 0))
    y, rep, _ = run_protected(plan, tw, torch.from_numpy(x).cuda(), Scheme.TWO_SIDED_GROUP,
                              injector=BitFlipInjector(spec))
    assert [c["signal"] for c in rep.corrected] == [9] and rel_l2(y, ref) < 1e-6
    with pytest.raises(NotImplementedError):
        big = fit_group_size(make_plan(1 << 16, "fp32", batch=16), 16)
        _lib.check(_lib.load().tfft_set_check_level(native_plan(big, torch.cuda.current_device()).handle, 1))
