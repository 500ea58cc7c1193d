"""Independent DFT check (reference ``fft_core/reference.py:1-39``).

``dft_reference`` evaluates y_j = sum_k x_k w^(jk) directly, for any length
n <= ORACLE_MAX_N, in complex128 on the GPU (``tfft_dft``: a kernel of its
own, one output per thread, exactly rounded w^m table). It shares nothing
with the Stockham kernels, which is what makes it a check of them. Host
inputs come back as numpy arrays (of the input's complex dtype, like the
reference), CUDA tensors as CUDA tensors.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _device, _lib

ORACLE_MAX_N = 2**14


def dft_reference(x, inverse: bool = False):
    """Direct evaluation of y_j = sum_n x_n w^(jn); inverse scales by 1/N.
    Batched inputs transform along the last axis (reference.py:12-39)."""
    dev_in = _device.is_device(x)
    if dev_in:
        xt = x
        single = xt.dim() == 1
        n = xt.shape[-1]
    else:
        xa = np.asarray(x)
        single = xa.ndim == 1
        n = xa.shape[-1]
    if n < 1:
        raise ValueError("empty signal")
    if n > ORACLE_MAX_N:
        raise ValueError(f"oracle limited to n <= {ORACLE_MAX_N}, got {n}")
    _device.require_cuda()
    if dev_in:
        xs = (xt.reshape(1, -1) if single else xt.reshape(-1, n)).to(torch.complex128).contiguous()
    else:
        xs, _ = _device.to_device(xa.reshape(1, -1) if single else xa.reshape(-1, n), np.complex128)
    out = torch.empty_like(xs)
    _lib.check(_lib.load().tfft_dft(xs.data_ptr(), out.data_ptr(), xs.shape[0], n, int(bool(inverse)),
                                    _device.stream_ptr()), "tfft_dft")
    if dev_in:
        res = out[0] if single else out.reshape(xt.shape)
        return res.to(xt.dtype) if xt.is_complex() else res
    res = out.cpu().numpy()
    res = res[0] if single else res.reshape(xa.shape)
    return res.astype(xa.dtype) if np.iscomplexobj(xa) else res
