"""Raw signal files: headerless little-endian interleaved (re, im) pairs
(reference ``signal_io.py:1-33``).

That byte format IS the complex64 / complex128 memory layout, so
``transform_file`` streams a file through the device without ever building a
host array: ``tfft_run_protected_file`` reads chunks of whole checksum groups
into pinned memory, copies them in, runs the fused protected transform,
copies them out and writes them, with every stage of different chunks in
flight at once. ``read_signals`` / ``write_signals`` are the reference's
host-side format helpers (file <-> numpy).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import _device, _lib

_REAL = {"fp32": np.dtype("<f4"), "fp64": np.dtype("<f8")}
_COMPLEX = {"fp32": np.dtype("<c8"), "fp64": np.dtype("<c16")}


def _check_precision(precision):
    if precision not in _REAL:
        raise ValueError("precision must be 'fp32' or 'fp64'")


def signal_count(path, n: int, precision: str = "fp32") -> int:
    """Signals in a raw file; ValueError "input length mismatch" otherwise
    (signal_io.py:14-21)."""
    _check_precision(precision)
    size = os.stat(Path(path)).st_size
    per = 2 * n * _REAL[precision].itemsize
    if size == 0 or size % per:
        raise ValueError(f"input length mismatch: {size} bytes is not a whole number of "
                         f"{n}-sample {precision} signals")
    return size // per


def read_signals(path, n: int, precision: str = "fp32") -> np.ndarray:
    """Load a (batch, n) complex array; batch is inferred from the file size."""
    batch = signal_count(path, n, precision)
    arr = np.fromfile(Path(path), dtype=_COMPLEX[precision])
    return arr.reshape(batch, n).astype(_COMPLEX[precision].newbyteorder("="), copy=False)


def write_signals(path, data, precision: str = "fp32") -> None:
    """Store a signal or batch as interleaved (re, im) pairs."""
    _check_precision(precision)
    if hasattr(data, "is_cuda") and data.is_cuda:
        data = data.cpu().numpy()
    arr = np.ascontiguousarray(np.asarray(data), dtype=_COMPLEX[precision]).reshape(-1)
    arr.tofile(Path(path))


def transform_file(input_path, output_path, n: int, precision: str = "fp32", scheme="none",
                   delta: float | None = None, inverse: bool = False, injector=None):
    """cli.py:54-67 ``transform`` as one streamed native call. Returns
    ``(RunReport, PassCounter, batch)``; the output file is written even when
    a group is unrecoverable (the report lists it)."""
    from .abft.encoding import EncodingKind, make_encoding
    from .abft.pipeline import DetectionConfig
    from .abft.protected import Scheme, _fault_struct, _report_buffers, default_delta, report_from_native
    from .fault_lab.bits import BitFlipInjector
    from .fft_core import PassCounter, fit_group_size, make_plan
    from .fft_core.plan import native_plan

    _device.require_cuda()
    batch = signal_count(input_path, n, precision)
    plan = fit_group_size(make_plan(n, precision, batch=batch), batch)
    scheme = Scheme(scheme)
    cfg = DetectionConfig(delta=delta if delta is not None else default_delta(precision))
    lib = _lib.load()
    h = native_plan(plan, _device.torch_current_device())
    td = _device.torch_dtype(plan.dtype)
    row = vals = None
    if scheme is not Scheme.NONE:
        enc = make_encoding(EncodingKind.WANG, n)
        row = enc.device_row(td, inverse)
        vals = enc.device_values(td)
    fault = None
    if injector is not None:
        if not isinstance(injector, BitFlipInjector):
            raise TypeError("transform_file takes a BitFlipInjector (or None)")
        if not injector.fired:
            fault = _fault_struct(injector)
    rep, bufs = _report_buffers(64, 64, 64)
    nb = ctypes.c_int64()
    _lib.check(lib.tfft_run_protected_file(
        h.handle, os.fsencode(str(input_path)), os.fsencode(str(output_path)),
        _lib.SCHEME_CODE[scheme.value], float(cfg.delta), float(cfg.abs_floor),
        _device.ptr(row), _device.ptr(vals), ctypes.byref(fault) if fault is not None else None,
        int(bool(inverse)), ctypes.byref(nb), ctypes.byref(rep), _device.stream_ptr()),
        "tfft_run_protected_file")
    if fault is not None and rep.fault_fired:
        injector.fired = True
    report = report_from_native(lib, h, rep, bufs, scheme, cfg.delta)
    counter = PassCounter(reads=report.pass_count // 2, writes=report.pass_count // 2)
    return report, counter, int(nb.value)
