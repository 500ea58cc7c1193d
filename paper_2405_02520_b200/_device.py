"""Device-buffer plumbing: numpy/torch inputs -> contiguous CUDA tensors.

Device (torch CUDA) inputs stay on the device and results are returned as
CUDA tensors. Host inputs (numpy arrays, CPU tensors, lists) are the
drop-in path of the reference's numpy API: they are staged through pinned
memory, transformed on the GPU and returned as numpy arrays of the plan's
dtype. Nothing is computed on the host.
"""

from __future__ import annotations

import numpy as np
import torch

_TORCH = {np.dtype(np.complex64): torch.complex64, np.dtype(np.complex128): torch.complex128}
_NUMPY = {torch.complex64: np.complex64, torch.complex128: np.complex128}


_CUDA_OK = False
_INIT = False


def require_cuda():
    # torch.cuda.is_available() re-reads the environment and NVML state on every
    # call (~10 us on the C1 latency path); once a device was seen, stay true
    global _CUDA_OK
    if _CUDA_OK:
        return
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2405_02520_b200 needs a CUDA device (there is no CPU fallback)")
    _CUDA_OK = True


def torch_dtype(np_dtype):
    return _TORCH[np.dtype(np_dtype)]


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, np_dtype, device=None):
    """Return (contiguous CUDA tensor of the plan dtype, input_was_host)."""
    require_cuda()
    td = torch_dtype(np_dtype)
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            t = x if x.dtype == td else x.to(td)
            return t.contiguous(), False
        host = x.to(td).contiguous()
    else:
        arr = np.ascontiguousarray(np.asarray(x), dtype=np_dtype)
        host = torch.from_numpy(arr)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if host.numel() * host.element_size() >= (1 << 20):
        if not host.is_pinned():
            host = host.pin_memory()
        return host.to(dev, non_blocking=True), True
    return host.to(dev), True


def is_host(x) -> bool:
    return not is_device(x)


def host_tensor(x, np_dtype) -> torch.Tensor:
    """Contiguous CPU tensor of the plan dtype sharing memory with `x` when it
    already has that dtype and layout (pinned CPU tensors stay pinned)."""
    td = torch_dtype(np_dtype)
    if isinstance(x, torch.Tensor):
        return x.to(td).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np_dtype))


def pinned_empty(shape, td) -> torch.Tensor:
    """Pinned host tensor from torch's caching host allocator."""
    return torch.empty(shape, dtype=td, pin_memory=True)


def to_host(t: torch.Tensor) -> np.ndarray:
    """D2H into pinned memory from torch's caching host allocator (no page
    faulting of fresh pageable memory per call); the numpy array keeps the
    pinned block alive and returns it to the cache when dropped."""
    if t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def torch_current_device() -> int:
    return torch._C._cuda_getDevice()


def stream_ptr():
    """The raw cudaStream_t of torch's current stream on the current device
    (the direct binding: torch.cuda.current_stream() builds a Stream object
    and re-checks availability on every call)."""
    global _INIT
    if not _INIT:
        torch.cuda.init()  # the raw bindings below assume an initialised CUDA state
        _INIT = True
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
