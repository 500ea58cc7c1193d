"""Transform execution (reference ``fft_core/execute.py:18-111``).

``fft_execute`` is one C-ABI call (``tfft_execute``): a single fused kernel
for n <= 2^13, otherwise one launch per reference stage with the four-step
transposes folded into the passes' address maps. ``PassCounter`` keeps the
reference's accounting contract — one read and one write sweep per stage —
which on the GPU is also the real HBM traffic of the launch sequence.

``on_stage`` hooks (fault injection with arbitrary callables) run the stages
one launch at a time and hand the hook a materialised copy of each
intermediate in the reference's layout, writing it back after the
hook returns. That is a test/debug path; ``BitFlipInjector`` faults are
injected inside the kernels instead (see abft/protected.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from .. import _device, _lib
from .plan import FftPlan, Stage, native_plan, validate_signal
from .twiddle import TwiddleTable

BACKENDS = ("auto", "cuda", "ext", "numpy")


@dataclass
class PassCounter:
    reads: int = 0
    writes: int = 0

    @property
    def total(self) -> int:
        return self.reads + self.writes


def check_backend(name: str):
    """The reference's backend names are accepted for signature compatibility
    (kernels/__init__.py:28-39); all of them run the single CUDA path."""
    if name not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}; available: {BACKENDS}")


# ---- pass layout <-> reference intermediate layout (for on_stage hooks)
def to_reference_layout(buf: torch.Tensor, plan: FftPlan, k: int) -> torch.Tensor:
    b, n = buf.shape
    dims = plan.dims
    if len(dims) == 1:
        return buf.clone()
    d0 = dims[0]
    if k == 0:
        return buf.view(b, d0, n // d0).transpose(1, 2).reshape(b, n)
    if len(dims) == 2:  # last of two: natural f = k0 + d0*k1 -> k0*d1 + k1
        return buf.view(b, dims[1], d0).transpose(1, 2).reshape(b, n)
    d1, d2 = dims[1], dims[2]
    if k == 1:  # [k0, k1, c2] -> [k0, c2, k1]
        return buf.view(b, d0, d1, d2).permute(0, 1, 3, 2).reshape(b, n)
    return buf.view(b, d2, d1, d0).permute(0, 3, 2, 1).reshape(b, n)


def from_reference_layout(ref: torch.Tensor, plan: FftPlan, k: int) -> torch.Tensor:
    b, n = ref.shape
    dims = plan.dims
    if len(dims) == 1:
        return ref
    d0 = dims[0]
    if k == 0:
        return ref.view(b, n // d0, d0).transpose(1, 2).reshape(b, n)
    if len(dims) == 2:
        return ref.view(b, d0, dims[1]).transpose(1, 2).reshape(b, n)
    d1, d2 = dims[1], dims[2]
    if k == 1:
        return ref.view(b, d0, d2, d1).permute(0, 1, 3, 2).reshape(b, n)
    return ref.view(b, d0, d1, d2).permute(0, 3, 2, 1).reshape(b, n)


def execute_device(plan: FftPlan, x: torch.Tensor, out: torch.Tensor | None = None,
                   inverse: bool = False) -> torch.Tensor:
    """(B, n) CUDA tensor -> new (B, n) CUDA tensor; one C-ABI call."""
    lib = _lib.load()
    if out is None:
        out = torch.empty_like(x)
    h = native_plan(plan, x.device.index)
    _lib.check(lib.tfft_execute(h.handle, x.data_ptr(), out.data_ptr(), x.shape[0],
                                int(bool(inverse)), _device.stream_ptr()), "tfft_execute")
    return out


def execute_staged(plan: FftPlan, x: torch.Tensor, inverse: bool, hook) -> torch.Tensor:
    """Stage-at-a-time execution with a reference-layout hook after each stage."""
    lib = _lib.load()
    h = native_plan(plan, x.device.index)
    batch = x.shape[0]
    work = x
    for k in range(len(plan.stages)):
        out = torch.empty_like(x)
        _lib.check(lib.tfft_execute_stage(h.handle, k, work.data_ptr(), out.data_ptr(), batch,
                                          int(bool(inverse)), _device.stream_ptr()),
                   "tfft_execute_stage")
        if hook is not None:
            ref = to_reference_layout(out, plan, k).contiguous()
            hook(k, ref)
            out = from_reference_layout(ref, plan, k).contiguous()
        work = out
    if inverse:
        _lib.check(lib.tfft_scale(work.data_ptr(), work.numel(), work.element_size(),
                                  1.0 / plan.n, _device.stream_ptr()), "tfft_scale")
    return work


def fft_execute(plan: FftPlan, twiddles: TwiddleTable, data, inverse: bool = False,
                counter: PassCounter | None = None, on_stage=None, backend: str = "auto"):
    """Transform a signal (1-D) or batch (2-D, signal-major) out-of-place.

    Device tensors in -> device tensor out; host arrays in -> numpy out.
    ``on_stage(k, view)`` is called after stage ``k`` with a mutable
    (batch, n) view in the reference's intermediate layout.
    """
    check_backend(backend)
    validate_signal(data, plan.n)
    if twiddles is not None and twiddles.n != plan.n:
        raise ValueError("twiddle table does not match the plan")
    x, host = _device.to_device(data, plan.dtype)
    single = x.dim() == 1
    x2 = x.reshape(-1, plan.n)
    if counter is None:
        counter = PassCounter()
    nst = len(plan.stages)
    counter.reads += nst
    counter.writes += nst
    if on_stage is None:
        y = execute_device(plan, x2, inverse=inverse)
    else:
        y = execute_staged(plan, x2, inverse, on_stage)
    y = y[0] if single else y
    return _device.to_host(y) if host else y


def stage_pass(buffer, stage: Stage, butterfly, counter: PassCounter, inverse: bool = False,
               inter=None, backend: str = "auto"):
    """One stage on its own (execute.py:28-53): tile DFTs of every row of
    ``buffer.reshape(-1, dim)`` plus the optional inter-stage factors.
    Compatibility utility; ``fft_execute`` does not go through it."""
    check_backend(backend)
    x, host = _device.to_device(buffer, np.asarray(butterfly).dtype
                                if not isinstance(butterfly, torch.Tensor)
                                else _np_dtype(butterfly.dtype))
    if x.numel() % stage.dim:
        raise ValueError(f"buffer size {x.numel()} not divisible by stage dim {stage.dim}")
    tiles = x.reshape(-1, stage.dim)
    counter.reads += 1
    out = torch.empty_like(tiles)
    lib = _lib.load()
    _lib.check(lib.tfft_tile_fft(tiles.data_ptr(), out.data_ptr(), tiles.shape[0], stage.dim,
                                 tiles.element_size(), int(bool(inverse)), 0,
                                 _device.stream_ptr()), "tfft_tile_fft")
    if inter is not None:
        f = torch.as_tensor(np.asarray(inter) if not isinstance(inter, torch.Tensor) else inter,
                            device=out.device, dtype=out.dtype)
        rest, dim = f.shape
        out.view(-1, rest, dim).mul_(f.conj() if inverse else f)
    counter.writes += 1
    out = out.reshape(x.shape)
    return _device.to_host(out) if host else out


def _np_dtype(td):
    return np.complex64 if td == torch.complex64 else np.complex128
