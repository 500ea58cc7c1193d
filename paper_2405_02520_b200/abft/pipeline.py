"""Group checksum state, detection and correction (reference ``abft/pipeline.py``).

These are the reference's per-group entry points — encode / detect / correct
on a (bs, n) group — each one a C-ABI call on device buffers. The fused
batch path (``run_protected``) does not go through them: there the same
arithmetic runs inside the FFT's own load/store passes. They serve the
reference's API, its tests, and arbitrary-callable fault injection.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _device, _lib
from ..fft_core.plan import FftPlan, fit_group_size, make_plan, native_plan
from .encoding import EncodingVector

# Guards for near-zero checksums, scaled by each signal's l1 mass (pipeline.py:16).
FLOOR_COEF = {"fp32": 1e-6, "fp64": 1e-12}


class UnrecoverableError(RuntimeError):
    """The single-error assumption or a correction check failed."""


class LocationError(RuntimeError):
    """The quotient test could not name a corrupted index."""


@dataclass
class DetectionConfig:
    delta: float
    abs_floor: float = 0.0

    def __post_init__(self):
        if self.delta <= 0:
            raise ValueError("delta must be positive")
        if self.abs_floor < 0:
            raise ValueError("abs_floor must be >= 0")


@dataclass
class PendingFault:
    signal_idx: int
    detected_discrepancy: float


@dataclass
class FlaggedSignal:
    signal_idx: int
    rel_discrepancy: float
    epsilon_estimate: complex


@dataclass
class DetectionReport:
    flagged: list[FlaggedSignal] = field(default_factory=list)
    corrected: list[int] = field(default_factory=list)
    unrecoverable: bool = False
    rel_discrepancies: np.ndarray | None = None


@dataclass
class ChecksumState:
    """Device-resident group state (pipeline.py:60-69)."""

    group_size: int
    s0: torch.Tensor        # sum_b x_b                        (n,)  plan dtype
    s1: torch.Tensor        # sum_b (b+1) x_b                  (n,)  complex128
    c_in: torch.Tensor      # (e^T W) x_b                      (bs,) plan dtype
    x_l1: torch.Tensor      # sum_k |x_bk|                      (bs,) real dtype
    r0: torch.Tensor | None = None
    r1: torch.Tensor | None = None
    pending: PendingFault | None = None


def _precision(t: torch.Tensor) -> str:
    return "fp32" if t.dtype == torch.complex64 else "fp64"


def _group_plan(n: int, precision: str, bs: int) -> FftPlan:
    return fit_group_size(make_plan(n, precision, batch=bs), bs)


def _as_group(xg):
    x, host = _device.to_device(xg, np.asarray(xg).dtype if not isinstance(xg, torch.Tensor)
                                else (np.complex64 if xg.dtype == torch.complex64 else np.complex128))
    if x.dim() != 2:
        raise ValueError("group must have shape (bs, n)")
    return x, host


def _sums(plan: FftPlan, g: torch.Tensor):
    lib = _lib.load()
    n = g.shape[1]
    s0 = torch.empty(n, dtype=g.dtype, device=g.device)
    s1 = torch.empty(n, dtype=torch.complex128, device=g.device)
    h = native_plan(plan, g.device.index)
    _lib.check(lib.tfft_encode_group(h.handle, g.data_ptr(), g.shape[0], None, s0.data_ptr(),
                                     s1.data_ptr(), None, None, _device.stream_ptr()),
               "tfft_encode_group")
    return s0, s1


def encode_group(xg, enc: EncodingVector, inverse: bool = False) -> ChecksumState:
    """Load-pass accumulations of one group (pipeline.py:72-85)."""
    x, _ = _as_group(xg)
    bs, n = x.shape
    if enc.n != n:
        raise ValueError("length mismatch between group and encoding")
    prec = _precision(x)
    plan = _group_plan(n, prec, bs)
    lib = _lib.load()
    h = native_plan(plan, x.device.index)
    rdt = torch.float32 if prec == "fp32" else torch.float64
    s0 = torch.empty(n, dtype=x.dtype, device=x.device)
    s1 = torch.empty(n, dtype=torch.complex128, device=x.device)
    c_in = torch.empty(bs, dtype=x.dtype, device=x.device)
    x_l1 = torch.empty(bs, dtype=rdt, device=x.device)
    row = enc.device_row(x.dtype, inverse)
    _lib.check(lib.tfft_encode_group(h.handle, x.data_ptr(), bs, row.data_ptr(), s0.data_ptr(),
                                     s1.data_ptr(), c_in.data_ptr(), x_l1.data_ptr(),
                                     _device.stream_ptr()), "tfft_encode_group")
    return ChecksumState(group_size=bs, s0=s0, s1=s1, c_in=c_in, x_l1=x_l1)


def finalize_group(state: ChecksumState, yg) -> None:
    """Store-pass combinations r0 = sum y_b, r1 = sum (b+1) y_b (pipeline.py:88-97).
    Kept for API parity; the reference never reads them afterwards."""
    y, _ = _as_group(yg)
    plan = _group_plan(y.shape[1], _precision(y), y.shape[0])
    state.r0, state.r1 = _sums(plan, y)


def detect(state: ChecksumState, outputs, enc: EncodingVector, cfg: DetectionConfig,
           precision: str = "fp64") -> DetectionReport:
    """Flag signals whose output checksum disagrees (pipeline.py:104-135)."""
    y, _ = _as_group(outputs)
    bs, n = y.shape
    plan = _group_plan(n, _precision(y), bs)
    lib = _lib.load()
    h = native_plan(plan, y.device.index)
    rdt = torch.float32 if y.dtype == torch.complex64 else torch.float64
    rel = torch.empty(bs, dtype=rdt, device=y.device)
    raw = torch.empty(bs, dtype=y.dtype, device=y.device)
    vals = enc.device_values(y.dtype)
    if precision not in FLOOR_COEF:
        raise KeyError(precision)
    _lib.check(lib.tfft_detect(h.handle, y.data_ptr(), bs, _device.ptr(vals),
                               state.c_in.data_ptr(), state.x_l1.data_ptr(), float(cfg.abs_floor),
                               FLOOR_COEF[precision], rel.data_ptr(), raw.data_ptr(),
                               _device.stream_ptr()), "tfft_detect")
    rel_h = rel.cpu().numpy()
    raw_h = raw.cpu().numpy()
    delta = rel_h.dtype.type(cfg.delta)
    rep = DetectionReport(rel_discrepancies=rel_h)
    for b in np.flatnonzero(rel_h > delta):
        eps = complex(raw_h[b]) if np.isfinite(raw_h[b]) else complex(np.inf)
        rep.flagged.append(FlaggedSignal(int(b), float(rel_h[b]), eps))
    rep.unrecoverable = len(rep.flagged) > 1
    return rep


def locate_quotient(u0, u1, abs_floor: float = 0.0, count: int | None = None) -> int:
    """round(u1/u0) - 1 index recovery (pipeline.py:138-161); host utility."""
    u0 = np.asarray(u0.cpu() if isinstance(u0, torch.Tensor) else u0)
    u1 = np.asarray(u1.cpu() if isinstance(u1, torch.Tensor) else u1)
    k = int(np.argmax(np.abs(u0)))
    if abs(u0[k]) <= abs_floor:
        raise LocationError("no dominant discrepancy component above the floor")
    q = u1[k] / u0[k]
    nearest = round(q.real)
    if abs(q - nearest) > 0.25:
        raise LocationError(f"quotient {q} too far from an integer")
    idx = nearest - 1
    if idx < 0 or (count is not None and idx >= count):
        raise LocationError(f"located index {idx} out of range")
    return idx


def correct_group(state: ChecksumState, outputs, flagged_idx: int, plan: FftPlan, twiddles,
                  enc: EncodingVector, cfg: DetectionConfig, inverse: bool = False):
    """y_f = W s0 - sum_{b != f} y_b, then re-verify (pipeline.py:164-192)."""
    y, host = _as_group(outputs)
    bs, n = y.shape
    lib = _lib.load()
    h = native_plan(plan, y.device.index)
    fixed = torch.empty(n, dtype=y.dtype, device=y.device)
    s0 = state.s0.to(y.dtype).contiguous()
    _lib.check(lib.tfft_correct_signal(h.handle, s0.data_ptr(), y.data_ptr(), bs, int(flagged_idx),
                                       fixed.data_ptr(), int(bool(inverse)), _device.stream_ptr()),
               "tfft_correct_signal")
    out = y.clone()
    out[flagged_idx] = fixed
    finalize_group(state, out)
    post = detect(state, out, enc, cfg, plan.precision)
    if post.flagged:
        raise UnrecoverableError(
            "post-correction residual above threshold; combination checksum corrupted")
    return _device.to_host(out) if host else out
