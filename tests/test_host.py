"""Host-side logic of the product (no GPU): planner, plans, twiddle host
arrays, fault specs, reports, backend registry, kernel-plan generator.
The oracle port (pinned to the reference by test_oracle.py) is the checker."""

import json
import math

import numpy as np
import pytest

from oracle import port as P
from paper_2405_02520_b200 import planner
from paper_2405_02520_b200.abft.pipeline import DetectionConfig
from paper_2405_02520_b200.abft.protected import RunReport, Scheme, default_delta
from paper_2405_02520_b200.fault_lab.bits import BitFlipInjector, FaultSpec, apply_fault, flip_bit
from paper_2405_02520_b200.fft_core import (FftPlan, Stage, all_factors, build_twiddles,
                                            fit_group_size, make_plan, validate_signal)
from paper_2405_02520_b200.fft_core.execute import check_backend


def test_select_parameters_matches_reference_rules():
    for e in range(1, 30):
        for batch in (1, 3, 8, 16, 1000):
            p = planner.select_parameters(2**e, batch)
            dims, radices, bs = P.choose(2**e, batch)
            assert (p.dims, p.radices, p.bs) == (dims, radices, bs)


def test_table_rows_and_stage_rule():
    assert planner.select_parameters(2**10).dims == (1024,)
    assert planner.select_parameters(2**17, 8).dims == (256, 512)
    assert planner.select_parameters(2**23, 16).dims == (256, 128, 256)
    for e in range(1, 30):
        n = 2**e
        assert planner.stage_count(n) == (1 if n <= 2**13 else 2 if n <= 2**22 else 3)


def test_make_plan_and_fit_group_size_match_oracle():
    for e in range(1, 26):
        for prec in ("fp32", "fp64"):
            for batch in (1, 6, 16, 24):
                ours = fit_group_size(make_plan(2**e, prec, batch=batch), batch)
                ref = P.shrink_bs(P.plan_for(2**e, prec, batch=batch), batch)
                assert ours.dims == ref.dims and ours.bs == ref.bs
                assert ours.twiddle_mode == ref.twiddle_mode
                assert tuple(s.thread_radix for s in ours.stages) == ref.radices
    assert len(make_plan(2**12, "fp64", max_tile=2**6).stages) == 2


def test_plan_validation():
    with pytest.raises(ValueError):
        make_plan(1000)
    with pytest.raises(ValueError):
        make_plan(2**30)
    with pytest.raises(ValueError):
        FftPlan(16, (Stage(4, 4),), 1, "fp32", "direct")
    with pytest.raises(ValueError):
        FftPlan(16, (Stage(16, 16),), 1, "fp16", "direct")
    with pytest.raises(ValueError):
        validate_signal(np.zeros(12))
    with pytest.raises(ValueError):
        validate_signal(np.zeros(16), 8)


@pytest.mark.parametrize("mode", ["direct", "precomputed", "recurrence"])
def test_twiddle_host_arrays_match_oracle(mode):
    for n, prec in ((8, "fp32"), (2**12, "fp64"), (2**14, "fp64"), (2**17, "fp32")):
        plan = make_plan(n, prec)
        ours = all_factors(build_twiddles(plan, mode=mode))
        ref = np.concatenate([a.ravel() for st in P.twiddles_for(P.plan_for(n, prec), mode=mode)
                              for a in st if a is not None])
        assert np.array_equal(ours, ref)


def test_twiddle_validation():
    plan = make_plan(16)
    with pytest.raises(ValueError):
        build_twiddles(plan, mode="bogus")
    with pytest.raises(ValueError):
        build_twiddles(plan, renorm_interval=0)
    tw = build_twiddles(make_plan(4, "fp64"))
    np.testing.assert_allclose(tw.base ** np.arange(4), [1, -1j, -1, 1j], atol=1e-12)


def test_flip_bit_kats_and_involution():
    assert flip_bit(np.float32(1.0), 31) == np.float32(-1.0)
    assert flip_bit(np.float32(1.0), 23) == np.float32(0.5)
    assert flip_bit(np.float64(1.0), 63) == -1.0
    rng = np.random.default_rng(0)
    for v in rng.standard_normal(50).astype(np.float32):
        for bit in (0, 13, 30, 31):
            assert flip_bit(flip_bit(v, bit), bit).tobytes() == v.tobytes()
    with pytest.raises(ValueError):
        flip_bit(np.float32(1.0), 32)


def test_host_apply_fault_and_injector():
    buf = np.zeros((2, 4), dtype=np.complex64)
    buf[1, 2] = 1 + 1j
    apply_fault(buf, 1, 2, "re", 31)
    assert buf[1, 2] == np.complex64(-1 + 1j)
    inj = BitFlipInjector(FaultSpec(0, 0, 0, "re", 31, stage="stage:1"))
    b = np.ones((1, 2), dtype=np.complex64)
    inj("stage:0", 0, b)
    assert b[0, 0].real == 1.0
    inj("stage:1", 0, b)
    assert b[0, 0].real == -1.0 and inj.fired
    inj("stage:1", 0, b)
    assert b[0, 0].real == -1.0


def test_fault_spec_validation():
    with pytest.raises(ValueError):
        FaultSpec(0, 0, 0, "xx", 1)
    with pytest.raises(ValueError):
        FaultSpec(0, 0, 0, "re", -1)


def test_report_json_schema_and_defaults():
    rep = RunReport(scheme="two_sided_group", delta=1e-4, groups=2)
    doc = json.loads(rep.to_json())
    assert set(doc) == {"scheme", "delta", "groups", "flagged", "corrected", "unrecoverable",
                        "recompute_count", "pass_count"}
    assert default_delta("fp32") == 1e-4 and default_delta("fp64") == 1e-9
    assert Scheme("two_sided_thread") is Scheme.TWO_SIDED_THREAD
    with pytest.raises(ValueError):
        DetectionConfig(delta=0.0)
    with pytest.raises(ValueError):
        DetectionConfig(delta=1e-4, abs_floor=-1)


def test_backend_names():
    for name in ("auto", "cuda", "ext", "numpy"):
        check_backend(name)
    with pytest.raises(ValueError):
        check_backend("opencl")
    from paper_2405_02520_b200.kernels import available_backends, get_backend
    assert available_backends() == ("cuda",)
    assert get_backend("auto").NAME == "cuda"
    with pytest.raises(ValueError):
        get_backend("numpy")


def test_codegen_configs_are_consistent():
    from paper_2405_02520_b200 import codegen
    for c in codegen.single_configs():
        assert math.prod(c["radices"]) == c["n"] and c["threads"] <= 1024
        assert c["smem"] <= 227 * 1024 and c["threads"] % 32 == 0
        assert all(c["e"] % r == 0 for r in c["radices"])
    for c in codegen.pass_configs():
        assert math.prod(c["radices"]) == c["l"] and c["threads"] <= 1024
        assert c["smem"] <= 227 * 1024 and c["threads"] % 32 == 0
    # the chosen smem padding is never worse than no padding
    for c in codegen.single_configs():
        if len(c["radices"]) > 1:
            eb = codegen.ELEM_BYTES[c["prec"]]
            assert (codegen.smem_cost(c["n"], c["e"], c["radices"], c["ps"], eb)
                    <= codegen.smem_cost(c["n"], c["e"], c["radices"], 0, eb))


def _cf_row(n, L, inverse):
    """A float64 restatement of the device's closed-form Wang row (multi.cuh:
    wang_col_base / the per-launch cot(j pi/L) table / the addition formula /
    the one Laurent-patched pole element per thread), for the first pass of
    an n-point transform with stage length L, one thread per (column, t) and
    E = 16 rows per thread (TPS = L / 16)."""
    n3, h = 3 * n, 3 * n // 2
    r0 = n // L
    E = min(16, L)
    tps = L // E
    kap = int(n3 * (1.0 / (256.0 * math.pi))) + 1
    cot = np.zeros(n)
    cj = np.array([0.0] + [(-1 if inverse else 1) * math.cos(math.pi * j / L) / math.sin(math.pi * j / L)
                           for j in range(1, L)])
    dk = (-3 if inverse else 3) * r0
    for lo in range(r0):
        kk = n - 3 * lo if inverse else n + 3 * lo
        kk = kk - n3 if kk > h else (kk + n3 if kk <= -h else kk)
        cc = math.cos(math.pi * kk / n3) / math.sin(math.pi * kk / n3)
        for t in range(tps):
            kt = kk + dk * t
            kt = kt - n3 if kt > h else (kt + n3 if kt <= -h else kt)
            dm = dk * tps
            ms = int(round(-kt / dm)) % E
            km = kt + dm * ms
            km = km - n3 if km > h else (km + n3 if km <= -h else km)
            pole = -kap < km < kap and (t + ms * tps) != 0
            for m in range(E):
                j = t + m * tps
                c = cc if j == 0 else (cc * cj[j] - 1.0) / (cc + cj[j])
                if pole and m == ms:
                    d = km * math.pi / n3
                    c = 1 / d - d * (1 / 3 + d * d * (1 / 45 + d * d * 2 / 945))
                cot[lo + j * r0] = c
    return cot


@pytest.mark.parametrize("n,L", [(1 << 12, 64), (1 << 14, 128), (1 << 16, 256)])
@pytest.mark.parametrize("inverse", [False, True])
def test_closed_form_etw_matches_reference_row(n, L, inverse):
    """The first pass's closed-form input-side checksum x . etw =
    (A/2)(S0 - i S1), S1 = sum x cot (A = 1 - w3^n, inverse / n), against the
    reference's FFT-computed row (abft/encoding.py:58-62 via the oracle)."""
    enc = P.encoding_for("wang", n, "c")
    row = enc.etw_inv if inverse else enc.etw
    cot = _cf_row(n, L, inverse)
    rng = np.random.default_rng([n, L])
    x = rng.standard_normal((4, n)) + 1j * rng.standard_normal((4, n))
    s0 = x.sum(axis=1)
    s1 = (x * cot).sum(axis=1)
    hs = 0.8660254037844386 * (1 if n % 3 == 1 else -1)
    g = 0.5 / n if inverse else 0.5
    cin = (s0.real + s1.imag + 1j * (s0.imag - s1.real)) * complex(1.5 * g, hs * g)
    ref = x @ row
    assert np.max(np.abs(cin - ref) / np.abs(ref)) < 1e-12
