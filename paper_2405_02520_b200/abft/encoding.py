"""Checksum encodings (reference ``abft/encoding.py:15-94``).

An encoding vector e gives the output checksum e^T y; its image e^T W (the
DFT of e, W being symmetric) predicts that checksum from the input. As in
the reference, e^T W and e^T W^-1 are computed with the package's own FFT —
here the fp64 GPU transform — and kept on the device, with per-dtype casts
cached for the fused kernels.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from .. import _device


class EncodingKind(str, Enum):
    WANG = "wang"
    JOU = "jou"
    ONES = "ones"
    LINEAR = "linear"


def _values(kind: EncodingKind, length: int) -> np.ndarray:
    k = np.arange(length)
    if kind is EncodingKind.WANG:
        return np.exp(-2j * np.pi / 3) ** (k % 3)
    if kind is EncodingKind.JOU:
        return np.exp(-2j * np.pi / length) ** k
    if kind is EncodingKind.ONES:
        return np.ones(length, dtype=np.complex128)
    if kind is EncodingKind.LINEAR:
        return (k + 1).astype(np.complex128)
    raise ValueError(f"unknown encoding kind {kind}")


@dataclass(frozen=True, eq=False)
class EncodingVector:
    """Weights e and transform-side rows, device-resident (complex128)."""

    kind: EncodingKind
    values_dev: torch.Tensor
    etw_dev: torch.Tensor
    etw_inv_dev: torch.Tensor
    requires_variant_input: bool = False
    _casts: dict = field(default_factory=dict, repr=False)

    # host views, for API compatibility with the reference's numpy fields
    @functools.cached_property
    def values(self) -> np.ndarray:
        return self.values_dev.cpu().numpy()

    @functools.cached_property
    def etw(self) -> np.ndarray:
        return self.etw_dev.cpu().numpy()

    @functools.cached_property
    def etw_inv(self) -> np.ndarray:
        return self.etw_inv_dev.cpu().numpy()

    @property
    def n(self) -> int:
        return int(self.values_dev.shape[0])

    def device_row(self, dtype: torch.dtype, inverse: bool = False) -> torch.Tensor:
        """e^T W (or e^T W^-1) cast to the transform dtype (pipeline.py:79)."""
        key = ("row", dtype, bool(inverse))
        t = self._casts.get(key)
        if t is None:
            t = (self.etw_inv_dev if inverse else self.etw_dev).to(dtype).contiguous()
            self._casts[key] = t
        return t

    def device_values(self, dtype: torch.dtype) -> torch.Tensor | None:
        """Output-side weights cast to dtype; None for Wang (computed in-kernel)."""
        if self.kind is EncodingKind.WANG:
            return None
        key = ("values", dtype)
        t = self._casts.get(key)
        if t is None:
            t = self.values_dev.to(dtype).contiguous()
            self._casts[key] = t
        return t


def _dft_small(values: np.ndarray, inverse: bool) -> np.ndarray:
    # Non-power-of-two lengths never reach the transform path (plans are
    # power-of-two); the reference falls back to its brute-force DFT there
    # (encoding.py:63-65) and so do we — setup-only, tiny.
    n = values.shape[0]
    sign = 1.0 if inverse else -1.0
    k = np.arange(n)
    w = np.exp(sign * 2j * np.pi * np.outer(k, k) / n)
    out = values @ w
    return out / n if inverse else out


@functools.lru_cache(maxsize=64)
def _make(kind: EncodingKind, length: int, device: int) -> EncodingVector:
    values = _values(kind, length)
    dev = torch.device("cuda", device)
    if length >= 2 and length & (length - 1) == 0:
        from ..fft_core import build_twiddles, fft_execute, make_plan
        plan = make_plan(length, precision="fp64")
        tw = build_twiddles(plan)
        v = torch.from_numpy(values).to(dev)
        etw = fft_execute(plan, tw, v)
        etw_inv = fft_execute(plan, tw, v, inverse=True)
    else:
        v = torch.from_numpy(values).to(dev)
        etw = torch.from_numpy(_dft_small(values, False)).to(dev)
        etw_inv = torch.from_numpy(_dft_small(values, True)).to(dev)
    return EncodingVector(kind=kind, values_dev=v, etw_dev=etw.contiguous(),
                          etw_inv_dev=etw_inv.contiguous(),
                          requires_variant_input=kind is EncodingKind.JOU)


def make_encoding(kind, length: int) -> EncodingVector:
    """Weights and their transform-side images for ``length`` (encoding.py:47-72)."""
    kind = EncodingKind(kind)
    if length < 1:
        raise ValueError("encoding length must be >= 1")
    _device.require_cuda()
    return _make(kind, int(length), _device.torch_current_device())


def jou_variant_input(x):
    """x'_k = 2 x_k + x_{(k+1) mod n} (encoding.py:75-80)."""
    if isinstance(x, torch.Tensor):
        if x.shape[-1] < 2:
            raise ValueError("variant input needs length >= 2")
        return 2 * x + torch.roll(x, -1, dims=-1)
    x = np.asarray(x)
    if x.shape[-1] < 2:
        raise ValueError("variant input needs length >= 2")
    return 2 * x + np.roll(x, -1, axis=-1)


def left_checksum(x, enc: EncodingVector, side: str = "input"):
    """(e^T W) x on the input side, e^T y on the output side (encoding.py:83-94)."""
    if side == "input":
        weights = enc.etw_dev
    elif side == "output":
        weights = enc.values_dev
    else:
        raise ValueError("side must be 'input' or 'output'")
    if x.shape[-1] != weights.shape[0]:
        raise ValueError("length mismatch between signal and encoding")
    if isinstance(x, torch.Tensor):
        return x.to(weights.device, torch.complex128) @ weights
    return np.asarray(x) @ weights.cpu().numpy()
