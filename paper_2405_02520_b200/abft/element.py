"""Element-level two-sided check on one radix tile (reference
``abft/element.py:1-92``).

Protects one r x B tile computation Y = W_r X (column j = one signal's
r-point slice): the row-side checksum (e^T W) X locates the corrupted column,
the transformed column combination W (X e) locates the row and yields the
correction applied in place. Both sides are computed on the device in
complex128 (``tfft_element_encode`` / ``tfft_element_verify``); the optional
``inject(y)`` hook sees the freshly transformed tile as a host array, like the
reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from .. import _device, _lib
from .encoding import EncodingVector
from .pipeline import DetectionConfig, UnrecoverableError

TILE_RADICES = (2, 4, 8, 16, 32)


@dataclass
class ElementReport:
    located: tuple[int, int] | None = None  # (row, col) of the fixed entry
    corrected: bool = False
    col_discrepancies: np.ndarray | None = None


def two_sided_element(r: int, tile, enc_row: EncodingVector, enc_col: EncodingVector,
                      cfg: DetectionConfig, inject=None):
    """Transform an r x B tile under element-level two-sided protection;
    returns ``(y, ElementReport)``, raises UnrecoverableError when several
    columns are flagged or the two sides disagree."""
    if r not in TILE_RADICES:
        raise ValueError(f"tile radix must be one of {TILE_RADICES}")
    x = np.asarray(tile, dtype=np.complex128)
    if x.ndim == 1:
        x = x[:, None]
    if x.shape[0] != r:
        raise ValueError(f"tile must have {r} rows")
    _device.require_cuda()
    lib = _lib.load()
    b = x.shape[1]
    dev = torch.device("cuda", torch.cuda.current_device())
    c128 = torch.complex128

    def put(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(dev)

    xd = put(x)
    etw_row = put(enc_row.etw[:r])
    vals_row = put(enc_row.values[:r])
    vals_col = put(enc_col.values[:b])
    y = torch.empty((r, b), dtype=c128, device=dev)
    row_in = torch.empty(b, dtype=c128, device=dev)
    xe = torch.empty(r, dtype=c128, device=dev)
    st = _device.stream_ptr()
    _lib.check(lib.tfft_element_encode(r, b, xd.data_ptr(), y.data_ptr(), etw_row.data_ptr(),
                                       vals_col.data_ptr(), row_in.data_ptr(), xe.data_ptr(), st),
               "tfft_element_encode")
    if inject is not None:
        yh = y.cpu().numpy()
        inject(yh)
        y.copy_(torch.from_numpy(yh))
    rel = torch.empty(b, dtype=torch.float64, device=dev)
    res = (ctypes.c_int32 * 3)()
    _lib.check(lib.tfft_element_verify(r, b, y.data_ptr(), row_in.data_ptr(), xe.data_ptr(),
                                       vals_row.data_ptr(), vals_col.data_ptr(), float(cfg.delta),
                                       float(cfg.abs_floor), rel.data_ptr(), res, st),
               "tfft_element_verify")
    report = ElementReport(col_discrepancies=rel.cpu().numpy())
    if res[0] == 2:
        raise UnrecoverableError("multiple corrupted columns in one tile")
    if res[0] == 3:
        raise UnrecoverableError("row/column disagreements inconsistent")
    out = y.cpu().numpy()
    if res[0] == 1:
        report.located = (int(res[1]), int(res[2]))
        report.corrected = True
    return out, report
