"""Protected batch execution (reference ``abft/protected.py:28-198``).

Fast path — no injector, or a ``BitFlipInjector``: one C-ABI call
(``tfft_run_protected``). The FFT kernels encode the per-signal input
checksums while loading, verify while storing, and append only flagged
signals; the host then reads a few bytes, decides per group exactly as the
reference does (>1 flag -> unrecoverable; ONE_SIDED recomputes the signal
from the clean input; TWO_SIDED_* rebuilds it as W s0 - sum of the healthy
outputs and re-verifies before committing). The bit flip of a
``BitFlipInjector`` is applied inside the kernels at the matching point.

Generic path — any other injector callable: group by group, the reference's
own sequence (encode on the pristine input, hook "input" on a working copy,
stage-at-a-time transform with "stage:<k>" hooks on reference-layout views,
hook "output", detect, correct) on device buffers.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from .. import _device, _lib
from ..fault_lab.bits import BitFlipInjector
from ..fft_core import FftPlan, PassCounter, TwiddleTable, fft_execute
from ..fft_core.execute import check_backend, execute_device, execute_staged
from ..fft_core.plan import native_plan
from .encoding import EncodingKind, EncodingVector, make_encoding
from .pipeline import (
    DetectionConfig,
    PendingFault,
    UnrecoverableError,
    correct_group,
    detect,
    encode_group,
    finalize_group,
)


class Scheme(str, Enum):
    NONE = "none"
    ONE_SIDED = "one_sided"
    TWO_SIDED_THREAD = "two_sided_thread"
    TWO_SIDED_GROUP = "two_sided_group"


@dataclass
class RunReport:
    scheme: str
    delta: float
    groups: int
    flagged: list[dict] = field(default_factory=list)
    corrected: list[dict] = field(default_factory=list)
    unrecoverable: list[int] = field(default_factory=list)
    recompute_count: int = 0
    pass_count: int = 0
    max_rel_discrepancy: float = 0.0

    def to_dict(self) -> dict:
        return {
            "scheme": self.scheme,
            "delta": self.delta,
            "groups": self.groups,
            "flagged": self.flagged,
            "corrected": self.corrected,
            "unrecoverable": self.unrecoverable,
            "recompute_count": self.recompute_count,
            "pass_count": self.pass_count,
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, separators=(",", ":"))


def default_delta(precision: str) -> float:
    return 1e-4 if precision == "fp32" else 1e-9


_WHERE = {"input": _lib.AT_INPUT, "output": _lib.AT_OUTPUT}


def _fault_struct(inj: BitFlipInjector) -> _lib.Fault | None:
    spec = inj.spec
    f = _lib.Fault()
    f.signal = spec.signal_idx
    f.element = spec.element_idx
    f.component = 0 if spec.component == "re" else 1
    f.bit = spec.bit
    if spec.stage in _WHERE:
        f.where, f.stage = _WHERE[spec.stage], 0
    elif spec.stage.startswith("stage:"):
        f.where, f.stage = _lib.AT_STAGE, int(spec.stage.split(":", 1)[1])
    else:  # a `where` the reference never emits: the injector never fires
        return None
    return f


def _report_buffers(cap_f, cap_c, cap_u):
    rep = _lib.Report()
    flags = (_lib.Flag * max(cap_f, 1))()
    cg = (ctypes.c_int64 * max(cap_c, 1))()
    cs = (ctypes.c_int64 * max(cap_c, 1))()
    ur = (ctypes.c_int64 * max(cap_u, 1))()
    rep.flagged, rep.flagged_cap = flags, cap_f
    rep.corrected_group, rep.corrected_signal, rep.corrected_cap = cg, cs, cap_c
    rep.unrecoverable, rep.unrecoverable_cap = ur, cap_u
    return rep, (flags, cg, cs, ur)


def report_from_native(lib, h, rep, bufs, scheme, delta) -> RunReport:
    """RunReport of a native call; lists longer than the first buffers (a
    degenerate batch) are re-read whole with tfft_report_fetch."""
    if (rep.n_flagged > rep.flagged_cap or rep.n_corrected > rep.corrected_cap
            or rep.n_unrecoverable > rep.unrecoverable_cap):
        full, bufs = _report_buffers(rep.n_flagged, rep.n_corrected, rep.n_unrecoverable)
        _lib.check(lib.tfft_report_fetch(h.handle, ctypes.byref(full)), "tfft_report_fetch")
    flags, cg, cs, ur = bufs
    report = RunReport(scheme=scheme.value, delta=delta, groups=int(rep.groups))
    report.flagged = [{"group": int(flags[i].group), "signal": int(flags[i].signal),
                       "discrepancy": float(flags[i].discrepancy)} for i in range(rep.n_flagged)]
    report.corrected = [{"group": int(cg[i]), "signal": int(cs[i])} for i in range(rep.n_corrected)]
    report.unrecoverable = [int(ur[i]) for i in range(rep.n_unrecoverable)]
    report.recompute_count = int(rep.recompute_count)
    report.pass_count = int(rep.pass_count)
    report.max_rel_discrepancy = float(rep.max_rel_discrepancy)
    return report


def _fused(plan, x, out, scheme, cfg, enc, inverse, injector, host=False):
    """One C-ABI call: tfft_run_protected on device tensors, or (host=True)
    tfft_run_protected_host streaming host tensors through the device."""
    lib = _lib.load()
    dev = torch.cuda.current_device() if host else x.device.index
    h = native_plan(plan, dev)
    batch = x.shape[0]
    rep, bufs = _report_buffers(64, 64, 64)
    fault = None
    if injector is not None and not injector.fired:
        fault = _fault_struct(injector)
    code = _lib.SCHEME_CODE[scheme.value]
    row = vals = None
    if scheme is not Scheme.NONE:
        row = enc.device_row(x.dtype, inverse)
        vals = enc.device_values(x.dtype)
    entry = lib.tfft_run_protected_host if host else lib.tfft_run_protected
    _lib.check(entry(
        h.handle, x.data_ptr() if batch else None, out.data_ptr() if batch else None, batch, code,
        float(cfg.delta), float(cfg.abs_floor), _device.ptr(row), _device.ptr(vals),
        ctypes.byref(fault) if fault is not None else None,
        int(bool(inverse)), ctypes.byref(rep), _device.stream_ptr()), "tfft_run_protected")
    if fault is not None and rep.fault_fired:
        injector.fired = True
    return report_from_native(lib, h, rep, bufs, scheme, cfg.delta)


def _generic(plan, twiddles, x, out, scheme, cfg, enc, inverse, injector, counter):
    """The reference's per-group sequence with an arbitrary injector callable."""
    bs = plan.bs
    report = RunReport(scheme=scheme.value, delta=cfg.delta, groups=x.shape[0] // bs)
    protected = scheme is not Scheme.NONE
    nst = len(plan.stages)
    for g, start in enumerate(range(0, x.shape[0], bs)):
        xg = x[start:start + bs]
        state = encode_group(xg, enc, inverse=inverse) if protected else None
        work = xg.clone()
        injector("input", start, work)

        def hook(k, view, _s=start):
            injector(f"stage:{k}", _s, view)

        yg = execute_staged(plan, work, inverse, hook)
        counter.reads += nst
        counter.writes += nst
        injector("output", start, yg)
        if not protected:
            out[start:start + bs] = yg
            continue
        finalize_group(state, yg)
        det = detect(state, yg, enc, cfg, plan.precision)
        report.max_rel_discrepancy = max(report.max_rel_discrepancy,
                                         float(np.max(det.rel_discrepancies, initial=0.0)))
        for f in det.flagged:
            report.flagged.append({"group": g, "signal": start + f.signal_idx,
                                   "discrepancy": f.rel_discrepancy})
        if det.unrecoverable or not det.flagged:
            if det.unrecoverable:
                report.unrecoverable.append(g)
            out[start:start + bs] = yg
            continue
        local = det.flagged[0].signal_idx
        if scheme is Scheme.ONE_SIDED:
            yg = yg.clone()
            yg[local] = execute_device(plan, xg[local:local + 1].contiguous(), inverse=inverse)[0]
            counter.reads += nst
            counter.writes += nst
            report.recompute_count += 1
            report.corrected.append({"group": g, "signal": start + local})
        else:
            if scheme is Scheme.TWO_SIDED_GROUP:
                state.pending = PendingFault(local, det.flagged[0].rel_discrepancy)
            try:
                yg = correct_group(state, yg, local, plan, twiddles, enc, cfg, inverse=inverse)
                state.pending = None
                report.corrected.append({"group": g, "signal": start + local})
            except UnrecoverableError:
                report.unrecoverable.append(g)
        out[start:start + bs] = yg
    report.pass_count = counter.total
    return report


def run_protected(plan: FftPlan, twiddles: TwiddleTable, batch, scheme=Scheme.TWO_SIDED_GROUP,
                  cfg: DetectionConfig | None = None, injector=None, enc: EncodingVector | None = None,
                  inverse: bool = False, backend: str = "auto"):
    """Transform a (B, n) batch under the chosen protection scheme.

    Returns ``(outputs, RunReport, PassCounter)`` like the reference; outputs
    are a CUDA tensor for device input and a numpy array for host input.
    """
    scheme = Scheme(scheme)
    check_backend(backend)
    if cfg is None:
        cfg = DetectionConfig(delta=default_delta(plan.precision))
    if _device.is_host(batch) and (injector is None or isinstance(injector, BitFlipInjector)):
        # host drop-in: H2D / fused transform / D2H streamed in chunks
        _device.require_cuda()
        xh = _device.host_tensor(batch, plan.dtype)
        if xh.dim() != 2 or xh.shape[1] != plan.n:
            raise ValueError("batch must have shape (B, n) with n == plan.n")
        if xh.shape[0] % plan.bs:
            raise ValueError(f"batch size {xh.shape[0]} not divisible by group size {plan.bs}")
        if enc is None and scheme is not Scheme.NONE:
            enc = make_encoding(EncodingKind.WANG, plan.n)
        out = _device.pinned_empty(xh.shape, xh.dtype)
        report = _fused(plan, xh, out, scheme, cfg, enc, inverse, injector, host=True)
        counter = PassCounter(reads=report.pass_count // 2, writes=report.pass_count // 2)
        return out.numpy(), report, counter
    x, host = _device.to_device(batch, plan.dtype)
    if x.dim() != 2 or x.shape[1] != plan.n:
        raise ValueError("batch must have shape (B, n) with n == plan.n")
    if x.shape[0] % plan.bs:
        raise ValueError(f"batch size {x.shape[0]} not divisible by group size {plan.bs}")
    if enc is None and scheme is not Scheme.NONE:
        enc = make_encoding(EncodingKind.WANG, plan.n)
    out = torch.empty_like(x)
    if injector is None or isinstance(injector, BitFlipInjector):
        report = _fused(plan, x, out, scheme, cfg, enc, inverse, injector)
        counter = PassCounter(reads=report.pass_count // 2, writes=report.pass_count // 2)
    else:
        counter = PassCounter()
        report = _generic(plan, twiddles, x, out, scheme, cfg, enc, inverse, injector, counter)
    return (_device.to_host(out) if host else out), report, counter


def calibrate_delta(plan: FftPlan, twiddles: TwiddleTable, trials: int = 64,
                    quantile: float = 0.999, seed: int = 0, margin: float = 10.0) -> float:
    """``margin`` x the fault-free tail of the relative discrepancy over
    ``trials`` seeded batches (protected.py:174-198), same seeds as the
    reference."""
    enc = make_encoding(EncodingKind.WANG, plan.n)
    xs = []
    for t in range(trials):
        rng = np.random.default_rng([seed, t])
        xs.append((rng.standard_normal((plan.bs, plan.n))
                   + 1j * rng.standard_normal((plan.bs, plan.n))).astype(plan.dtype))
    discs = []
    cfg = DetectionConfig(delta=1e30)
    for x in xs:
        _, rep, _ = run_protected(plan, twiddles, x, Scheme.TWO_SIDED_GROUP, cfg, enc=enc)
        discs.append(rep.max_rel_discrepancy)
    return margin * float(np.quantile(np.asarray(discs), quantile))
