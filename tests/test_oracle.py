"""The oracle (oracle/port.py + oracle/stockham.c) pinned against the REAL
reference: golden vectors produced by tests/golden/make_golden.py and the
reference's own known-answer tests. CPU only."""

import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, random_batch, rel_l2
from golden.make_golden import fft_input, protected_input

GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       capture_output=True)


@pytest.fixture(scope="session")
def P():
    from oracle import port
    return port


def test_fft_bit_identical_to_reference(P):
    g = np.load(os.path.join(GOLD, "fft.npz"))
    for prec, exps in (("fp32", range(1, 15)), ("fp64", range(1, 16))):
        for e in exps:
            x = fft_input(prec, e)
            plan = P.plan_for(2**e, prec)
            tw = P.twiddles_for(plan)
            y = P.execute(plan, tw, x)
            assert np.array_equal(y.view(np.uint8), g[f"{prec}_{e}_y"].view(np.uint8)), (prec, e)
            if e <= 12:
                yi = P.execute(plan, tw, x, inverse=True)
                assert np.array_equal(yi.view(np.uint8), g[f"{prec}_{e}_yi"].view(np.uint8))


def test_encodings_match_reference(P):
    g = np.load(os.path.join(GOLD, "encodings.npz"))
    for kind in ("wang", "ones", "jou", "linear"):
        for n in (2, 4, 16, 1024):
            enc = P.encoding_for(kind, n)
            np.testing.assert_array_equal(enc.values, g[f"{kind}_{n}_values"])
            np.testing.assert_array_equal(enc.etw, g[f"{kind}_{n}_etw"])
            np.testing.assert_array_equal(enc.etw_inv, g[f"{kind}_{n}_etw_inv"])


def _case_injector(P, c):
    if c["fault"] is None:
        return None
    s, el, comp, bit, stage = c["fault"]
    return P.OneShot(s, el, comp, bit, stage)


def test_protected_runs_match_reference(P):
    cases = json.load(open(os.path.join(GOLD, "protected.json")))
    arrays = np.load(os.path.join(GOLD, "protected.npz"))
    for c in cases:
        x = protected_input(c["id"], c["n"], c["batch"], c["precision"])
        plan = P.shrink_bs(P.plan_for(c["n"], c["precision"], batch=c["batch"]), c["batch"])
        assert list(plan.dims) == c["dims"] and plan.bs == c["bs"]
        tw = P.twiddles_for(plan)
        inj = _case_injector(P, c)
        out, rep, cnt = P.protected(plan, tw, x, c["scheme"],
                                    delta=P.default_delta(c["precision"]), injector=inj,
                                    inverse=c["inverse"])
        assert json.loads(P.report_json(rep)) == c["report"], c["id"]
        assert rep["max_rel_discrepancy"] == c["max_rel"]
        assert cnt.total == c["pass_total"]
        if f"c{c['id']}_y" in arrays:
            assert np.array_equal(out.view(np.uint8), arrays[f"c{c['id']}_y"].view(np.uint8))


# ---- known-answer tests the reference's own suite pins (tests/test_fft_core.py etc.)
def test_kat_delta_and_constant(P):
    plan = P.plan_for(4, "fp64")
    tw = P.twiddles_for(plan)
    x = np.zeros(4, np.complex128)
    x[0] = 1
    np.testing.assert_allclose(P.execute(plan, tw, x), np.ones(4), atol=1e-12)
    np.testing.assert_allclose(P.execute(plan, tw, np.ones(4, np.complex128)), [4, 0, 0, 0],
                               atol=1e-12)


def test_kat_radix2_butterfly(P):
    out = P.tile_fft(np.array([[3.0 + 1j, 1.0 - 2j]]), np.array([1.0 + 0j]))
    np.testing.assert_allclose(out.ravel(), [4.0 - 1j, 2.0 + 3j], atol=1e-12)


def test_kat_flip_bit(P):
    assert P.flip(np.float32(1.0), 31) == np.float32(-1.0)
    assert P.flip(np.float32(1.0), 23) == np.float32(0.5)
    assert P.flip(np.float64(1.0), 63) == -1.0


def test_kat_wang_values(P):
    w3 = np.exp(-2j * np.pi / 3)
    np.testing.assert_allclose(P.encoding_values("wang", 4), [1, w3, w3**2, 1], atol=1e-12)


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("fp64", 1e-10)])
def test_oracle_vs_brute_force_dft(P, prec, tol):
    rng = np.random.default_rng(5)
    for e in (1, 3, 7, 10, 12):
        x = random_batch(rng, (2, 2**e), P.DTYPE[prec])
        plan = P.plan_for(2**e, prec)
        assert rel_l2(P.execute(plan, P.twiddles_for(plan), x), P.dft_oracle(x)) <= tol


def test_ref_kernel_matches_c_restatement(P):
    if not P.have_ref_kernel():
        pytest.skip("oracle/_ref not built (reference absent)")
    rng = np.random.default_rng(9)
    for length in (2, 64, 4096):
        for dt in (np.complex64, np.complex128):
            t = random_batch(rng, (3, length), dt)
            base = np.exp(-2j * np.pi * np.arange(length // 2) / length).astype(dt)
            a = P.tile_fft(t, base, kernel="c")
            b = P.tile_fft(t, base, kernel="ref")
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
