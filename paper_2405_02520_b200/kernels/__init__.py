"""The reference's backend plugin point (kernels/__init__.py:28-39), CUDA only.

``get_backend("cuda")`` (also returned for "auto") exposes ``tile_fft`` with
the reference's contract (kernels/_stockham.pyx:46-65): unscaled
natural-order DFT of every row of a (T, L) complex64/complex128 array, input
not mutated, inverse conjugates. It runs on the B200 through
``tfft_tile_fft``; host arrays are copied in and out. There is no numpy or
CPU backend: asking for one raises, like any unknown name.
"""

from __future__ import annotations

import os
import types

import numpy as np
import torch

from .. import _device, _lib

HAVE_EXT = True

# |base - w_L^k| bound for a factor table to count as the DFT's own (the
# reference builds it with np.exp in fp64 and casts to the plan dtype, or by
# the renormalised recurrence: <= ~1e-7 / 1e-14 away)
_BASE_TOL = {8: 1e-5, 16: 1e-12}


def _check_base(base, length, itemsize):
    """The kernels apply the exactly rounded roots w_L^k; a `base` that is not
    that table (within rounding) would ask for a different transform, so it
    is rejected instead of silently ignored (_stockham.pyx:32 multiplies by
    base[q * stride])."""
    if base is None:
        return
    b = base.detach().cpu().numpy() if isinstance(base, torch.Tensor) else np.asarray(base)
    half = length // 2
    if b.shape != (half,):
        raise ValueError("base must hold L/2 factors")
    if half == 0:
        return
    std = np.exp(-2j * np.pi * np.arange(half) / length)
    with np.errstate(all="ignore"):
        err = np.abs(b.astype(np.complex128) - std)
    if not np.all(err <= _BASE_TOL[itemsize]):
        raise ValueError("base must be the DFT factor table w_L^k = exp(-2 pi i k / L), k < L/2 "
                         "(this backend computes the DFT; other factor tables are not supported)")


def tile_fft(tiles, base=None, inverse: bool = False):
    if isinstance(tiles, torch.Tensor) and tiles.is_cuda:
        if tiles.dtype not in (torch.complex64, torch.complex128):
            raise TypeError(f"unsupported dtype {tiles.dtype}")
        _check_base(base, tiles.shape[-1], tiles.element_size())
        x = tiles.contiguous()
        out = torch.empty_like(x)
        t, length = x.shape
        _lib.check(_lib.load().tfft_tile_fft(x.data_ptr(), out.data_ptr(), t, length,
                                             x.element_size(), int(bool(inverse)), 0,
                                             _device.stream_ptr()), "tfft_tile_fft")
        return out
    arr = np.ascontiguousarray(tiles)
    if arr.dtype not in (np.complex64, np.complex128):
        raise TypeError(f"unsupported dtype {arr.dtype}")
    t, length = arr.shape
    _check_base(base, length, arr.dtype.itemsize)
    out = np.empty_like(arr)
    _device.require_cuda()
    _lib.check(_lib.load().tfft_tile_fft(arr.ctypes.data, out.ctypes.data, t, length,
                                         arr.dtype.itemsize, int(bool(inverse)), 1,
                                         _device.stream_ptr()), "tfft_tile_fft")
    return out


cuda_backend = types.SimpleNamespace(NAME="cuda", tile_fft=tile_fft)
_BACKENDS = {"cuda": cuda_backend}


def available_backends():
    return tuple(sorted(_BACKENDS))


def get_backend(name: str = "auto"):
    if name == "auto":
        name = os.environ.get("FFTSHIELD_BACKEND", "auto")
    if name == "auto":
        name = "cuda"
    try:
        return _BACKENDS[name]
    except KeyError:
        raise ValueError(f"unknown backend {name!r}; available: {available_backends()}") from None
