"""ORACLE — CPU restatement of the reference fault-tolerant FFT path.

Test infrastructure, not product code. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module, and only as the checker / the
CPU baseline. The product (``paper_2405_02520_b200``) never imports it.

It restates, function by function, the reference package ``fftshield``
(``/root/reference/pkg/src/fftshield``) hot path: the planner, twiddle
tables, the staged four-step driver, the Wang encoding, the checksum
pipeline (encode / detect / correct) and the protected runner, plus the
bit-flip injector. The radix-2 butterfly loop is the C restatement in
``oracle/stockham.c`` (built to ``oracle/liboracle.so``); when the
reference's own Cython kernel has been compiled into ``oracle/_ref/`` it can
be selected instead (``kernel="ref"``), which makes the hot loop literally
the reference's machine code.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference (in
this container only) and commits its outputs as fixtures;
``tests/test_oracle.py`` checks this port against them bit-for-bit.
"""

from __future__ import annotations

import ctypes
import glob
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# --------------------------------------------------------------------------
# butterfly kernel (kernels/_stockham.pyx:46-65 / kernels/numpy_backend.py)
# --------------------------------------------------------------------------

_C_LIB = None
_REF_EXT = None


def _c_lib():
    global _C_LIB
    if _C_LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/liboracle.so missing: run `make -C oracle`")
        lib = ctypes.CDLL(path)
        lib.oracle_tile_fft.restype = ctypes.c_int
        lib.oracle_tile_fft.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int]
        _C_LIB = lib
    return _C_LIB


def _ref_ext():
    """The reference's own compiled `_stockham` (built by oracle/build_ref.sh)."""
    global _REF_EXT
    if _REF_EXT is None:
        hits = glob.glob(os.path.join(_HERE, "_ref", "_stockham*.so"))
        if not hits:
            return None
        import importlib.machinery
        import importlib.util
        loader = importlib.machinery.ExtensionFileLoader("_stockham", hits[0])
        spec = importlib.util.spec_from_file_location("_stockham", hits[0], loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _REF_EXT = mod
    return _REF_EXT


def have_ref_kernel() -> bool:
    return _ref_ext() is not None


def tile_fft(tiles, base, inverse=False, kernel="c"):
    """Radix-2 Stockham over every row (_stockham.pyx:46-65)."""
    if kernel == "ref":
        ext = _ref_ext()
        if ext is None:
            raise RuntimeError("oracle/_ref/_stockham*.so not built")
        return ext.tile_fft(tiles, base, inverse)
    if kernel == "numpy":
        return _tile_fft_numpy(tiles, base, inverse)
    tiles = np.ascontiguousarray(tiles)
    if tiles.dtype not in (np.complex64, np.complex128):
        raise TypeError(f"unsupported dtype {tiles.dtype}")
    t, length = tiles.shape
    out = np.empty_like(tiles)
    base = np.ascontiguousarray(base, dtype=tiles.dtype)
    rc = _c_lib().oracle_tile_fft(tiles.ctypes.data, out.ctypes.data, t, length,
                                  base.ctypes.data, int(bool(inverse)),
                                  tiles.dtype.itemsize)
    if rc:
        raise ValueError("oracle_tile_fft: bad argument")
    return out


def _tile_fft_numpy(tiles, base, inverse=False):
    """numpy_backend.py:12-40 — same schedule, vectorised over tiles."""
    t, length = tiles.shape
    cur = np.array(tiles, order="C", copy=True)
    if length == 1:
        return cur
    nxt = np.empty_like(cur)
    half, span = length // 2, 1
    while half >= 1:
        w = base[:: length // (2 * span)][:span]
        if inverse:
            w = np.conj(w)
        src = cur.reshape(t, 2 * half, span)
        hi = src[:, half:, :] * w[None, None, :]
        dst = nxt.reshape(t, half, 2, span)
        dst[:, :, 0, :] = src[:, :half, :] + hi
        dst[:, :, 1, :] = src[:, :half, :] - hi
        cur, nxt = nxt, cur
        half //= 2
        span *= 2
    return cur


# --------------------------------------------------------------------------
# planner (planner.py:17-116) and plan (fft_core/plan.py:12-116)
# --------------------------------------------------------------------------

DTYPE = {"fp32": np.complex64, "fp64": np.complex128}
RDTYPE = {"fp32": np.float32, "fp64": np.float64}
EXEC_CAP = 2**22          # fft_core/plan.py:12 (MAX_SIGNAL_N)
BATCH_CAP = 1024          # fft_core/plan.py:13
TILE_CAP = 2**13          # fft_core/plan.py:14
RADICES = (2, 4, 8, 16, 32)  # planner.py:17
TUNED = {                 # planner.py:66-70 — (dims, radices, bs)
    2**10: ((1024,), (8,), 1),
    2**17: ((256, 512), (16, 16), 8),
    2**23: ((256, 128, 256), (16, 16, 16), 16),
}


def _log2_checked(n):
    if n < 2 or n & (n - 1):
        raise ValueError(f"size must be a power of two, got {n}")
    e = n.bit_length() - 1
    if not 1 <= e <= 29:
        raise ValueError(f"size 2^{e} outside supported range")
    return e


def n_stages(n):
    """planner.py:82-89: <=2^13 one stage, <=2^22 two, else three."""
    _log2_checked(n)
    return 1 if n <= 2**13 else (2 if n <= 2**22 else 3)


def split_even(n, count):
    """planner.py:92-97: balanced exponent split, larger parts last."""
    q, r = divmod(_log2_checked(n), count)
    return tuple(2**e for e in [q] * (count - r) + [q + 1] * r)


def choose(n, batch=1):
    """planner.py:104-116 -> (dims, radices, bs)."""
    _log2_checked(n)
    if batch < 1:
        raise ValueError("batch must be >= 1")
    if n in TUNED:
        return TUNED[n]
    dims = split_even(n, n_stages(n))
    return dims, tuple(min(16, d) for d in dims), min(max(batch, 1), 16)


@dataclass(frozen=True)
class Plan:
    n: int
    dims: tuple
    radices: tuple
    bs: int
    precision: str
    twiddle_mode: str

    @property
    def dtype(self):
        return DTYPE[self.precision]


def plan_for(n, precision="fp32", max_tile=TILE_CAP, batch=1, twiddle_mode=None):
    """fft_core/plan.py:64-91."""
    dims, radices, bs = choose(n, batch)
    if max_tile != TILE_CAP or max(dims) > max_tile:
        count = len(dims)
        while count <= 3 and max(split_even(n, count)) > max_tile:
            count += 1
        if count > 3:
            raise ValueError("cannot tile in 3 stages")
        if count != len(dims) or max(dims) > max_tile:
            dims = split_even(n, count)
            radices = tuple(min(16, d) for d in dims)
    mode = twiddle_mode or ("precomputed" if precision == "fp64" else "direct")
    return Plan(n, tuple(dims), tuple(radices), bs, precision, mode)


def shrink_bs(plan, batch):
    """fft_core/plan.py:94-101."""
    bs = plan.bs
    while batch % bs:
        bs -= 1
    return Plan(plan.n, plan.dims, plan.radices, bs, plan.precision, plan.twiddle_mode)


# --------------------------------------------------------------------------
# twiddles (fft_core/twiddle.py:18-105)
# --------------------------------------------------------------------------

def _seq_direct(count, m, dtype):
    return np.exp(-2j * np.pi * np.arange(count) / m).astype(dtype)


def _seq_recur(count, m, interval, dtype):
    step = complex(np.exp(-2j * np.pi / m))
    out = np.empty(count, dtype=np.complex128)
    cur = 1.0 + 0.0j
    for k in range(count):
        out[k] = cur
        cur *= step
        if (k + 1) % interval == 0:
            cur /= abs(cur)
    return out.astype(dtype)


def _glue(rows, cols, mode, interval, dtype):
    m = rows * cols
    if mode == "recurrence":
        gen = _seq_recur(cols, m, interval, np.complex128)
        out = np.empty((rows, cols), dtype=np.complex128)
        out[0] = 1.0
        for r in range(1, rows):
            out[r] = out[r - 1] * gen
            if r % interval == 0:
                out[r] /= np.abs(out[r])
        return out.astype(dtype)
    return np.exp(-2j * np.pi * np.outer(np.arange(rows), np.arange(cols)) / m).astype(dtype)


def twiddles_for(plan, mode=None, interval=16):
    """List of (butterfly, inter-or-None) per stage."""
    mode = mode or plan.twiddle_mode
    dtype = plan.dtype
    out = []
    for k, d in enumerate(plan.dims):
        if mode == "recurrence":
            bf = _seq_recur(max(d // 2, 1), d, interval, dtype)
        else:
            bf = _seq_direct(max(d // 2, 1), d, dtype)
        inter = None
        if k < len(plan.dims) - 1:
            rest = math.prod(plan.dims[k + 1:])
            inter = _glue(rest, d, mode, interval, dtype)
        out.append((bf, inter))
    return out


# --------------------------------------------------------------------------
# staged execution (fft_core/execute.py:28-111)
# --------------------------------------------------------------------------

@dataclass
class Passes:
    reads: int = 0
    writes: int = 0

    @property
    def total(self):
        return self.reads + self.writes


def _one_stage(buf, dim, bf, counter, inverse, inter, kernel):
    """execute.py:28-53."""
    tiles = buf.reshape(-1, dim)
    counter.reads += 1
    out = tile_fft(tiles, bf, inverse, kernel)
    if inter is not None:
        rest, d = inter.shape
        out.reshape(-1, rest, d)[:] *= (np.conj(inter) if inverse else inter)
    counter.writes += 1
    return out.reshape(buf.shape)


def _recurse(x, plan, tw, k, inverse, counter, hook, batch, kernel):
    """execute.py:82-106 — transpose, stage, transpose, recurse, transpose back."""
    rows, m = x.shape
    dim = plan.dims[k]
    bf, inter = tw[k]
    if k == len(plan.dims) - 1:
        if m != dim:
            raise ValueError("plan stage dims inconsistent with buffer")
        y = _one_stage(x, dim, bf, counter, inverse, None, kernel)
        if hook is not None:
            hook(k, y.reshape(batch, -1))
        return y
    rest = m // dim
    tiles = np.ascontiguousarray(x.reshape(rows, dim, rest).transpose(0, 2, 1))
    y = _one_stage(tiles.reshape(rows * rest, dim), dim, bf, counter, inverse, inter, kernel)
    if hook is not None:
        hook(k, y.reshape(batch, -1))
    z = np.ascontiguousarray(y.reshape(rows, rest, dim).transpose(0, 2, 1))
    u = _recurse(z.reshape(rows * dim, rest), plan, tw, k + 1, inverse, counter, hook,
                 batch, kernel)
    return np.ascontiguousarray(u.reshape(rows, dim, rest).transpose(0, 2, 1)).reshape(rows, m)


def check_signal(x, n=None, cap=EXEC_CAP):
    """fft_core/plan.py:104-116."""
    x = np.asarray(x)
    length = x.shape[-1]
    if length < 2 or length & (length - 1):
        raise ValueError(f"signal length must be a power of two, got {length}")
    if length > cap:
        raise ValueError(f"signal length {length} exceeds cap {cap}")
    if n is not None and length != n:
        raise ValueError(f"signal length {length} does not match plan size {n}")
    if x.ndim == 2 and not 1 <= x.shape[0] <= BATCH_CAP:
        raise ValueError(f"batch size must be in 1..{BATCH_CAP}")
    return x


def execute(plan, tw, data, inverse=False, counter=None, hook=None, kernel="c",
            cap=EXEC_CAP):
    """execute.py:56-79 — out-of-place, natural order, 1/N on inverse."""
    x = check_signal(data, plan.n, cap)
    single = x.ndim == 1
    work = np.ascontiguousarray(x, dtype=plan.dtype).reshape(-1, plan.n)
    counter = counter if counter is not None else Passes()
    out = _recurse(work, plan, tw, 0, inverse, counter, hook, work.shape[0], kernel)
    if inverse:
        out = out * plan.dtype(1.0 / plan.n)
    return out[0] if single else out


def dft_oracle(x, inverse=False):
    """fft_core/reference.py:12-39 — O(N^2) complex128 DFT, n <= 2^14."""
    x = np.asarray(x)
    xs = x.reshape(1, -1) if x.ndim == 1 else x
    n = xs.shape[-1]
    if n < 1 or n > 2**14:
        raise ValueError("oracle size out of range")
    sign = 1.0 if inverse else -1.0
    powers = np.exp(sign * 2j * np.pi * np.arange(n) / n)
    xc = xs.astype(np.complex128)
    out = np.empty_like(xc)
    cols = np.arange(n)
    block = max(1, 2**21 // n)
    for s in range(0, n, block):
        rows = np.arange(s, min(s + block, n))
        out[:, rows] = xc @ powers[(rows[:, None] * cols[None, :]) % n].T
    if inverse:
        out /= n
    res = out[0] if x.ndim == 1 else out
    return res.astype(x.dtype) if np.iscomplexobj(x) else res


# --------------------------------------------------------------------------
# encodings (abft/encoding.py:32-72)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Encoding:
    kind: str
    values: np.ndarray
    etw: np.ndarray
    etw_inv: np.ndarray


def encoding_values(kind, length):
    k = np.arange(length)
    if kind == "wang":
        return np.exp(-2j * np.pi / 3) ** (k % 3)
    if kind == "jou":
        return np.exp(-2j * np.pi / length) ** k
    if kind == "ones":
        return np.ones(length, dtype=np.complex128)
    if kind == "linear":
        return (k + 1).astype(np.complex128)
    raise ValueError(f"unknown encoding kind {kind}")


def encoding_for(kind, length, kernel="c"):
    values = encoding_values(kind, length)
    if length >= 2 and length & (length - 1) == 0:
        p = plan_for(length, "fp64")
        tw = twiddles_for(p)
        etw = execute(p, tw, values, kernel=kernel, cap=2**29)
        etw_inv = execute(p, tw, values, inverse=True, kernel=kernel, cap=2**29)
    else:
        etw = dft_oracle(values)
        etw_inv = dft_oracle(values, inverse=True)
    return Encoding(kind, values, np.asarray(etw, np.complex128),
                    np.asarray(etw_inv, np.complex128))


# --------------------------------------------------------------------------
# checksum pipeline (abft/pipeline.py:16-192)
# --------------------------------------------------------------------------

FLOOR = {"fp32": 1e-6, "fp64": 1e-12}


class Unrecoverable(RuntimeError):
    pass


@dataclass
class GroupState:
    bs: int
    s0: np.ndarray
    s1: np.ndarray
    c_in: np.ndarray
    x_l1: np.ndarray


def encode(xg, enc, inverse=False):
    """pipeline.py:72-85."""
    bs = xg.shape[0]
    wts = np.arange(1, bs + 1, dtype=np.float64)
    row = enc.etw_inv if inverse else enc.etw
    return GroupState(bs, xg.sum(axis=0), (wts[:, None] * xg).sum(axis=0),
                      xg @ row.astype(xg.dtype), np.abs(xg).sum(axis=1))


def verify(state, yg, enc, delta, abs_floor, precision):
    """pipeline.py:104-135 -> (flagged list of (idx, rel, eps), rel, unrecoverable)."""
    with np.errstate(all="ignore"):
        c_out = yg @ enc.values.astype(yg.dtype)
        raw = state.c_in - c_out
        floors = np.maximum(abs_floor, FLOOR[precision] * state.x_l1)
        rel = np.abs(raw) / np.maximum(np.abs(state.c_in), floors)
        bad = ~np.isfinite(yg).all(axis=1)
        rel = np.where(bad | ~np.isfinite(rel), np.inf, rel)
    flagged = [(int(b), float(rel[b]),
                complex(raw[b]) if np.isfinite(raw[b]) else complex(np.inf))
               for b in np.flatnonzero(rel > delta)]
    return flagged, rel, len(flagged) > 1


def repair(state, yg, f, plan, tw, enc, delta, abs_floor, inverse=False, kernel="c"):
    """pipeline.py:164-192 — y_f = W s0 - sum of the healthy outputs, re-verify."""
    ws0 = execute(plan, tw, state.s0, inverse=inverse, kernel=kernel, cap=2**29)
    others = np.delete(yg, f, axis=0).sum(axis=0)
    fixed = yg.copy()
    fixed[f] = ws0 - others
    post, _, _ = verify(state, fixed, enc, delta, abs_floor, plan.precision)
    if post:
        raise Unrecoverable("post-correction residual above threshold")
    return fixed


# --------------------------------------------------------------------------
# protected runner (abft/protected.py:63-171)
# --------------------------------------------------------------------------

def default_delta(precision):
    return 1e-4 if precision == "fp32" else 1e-9


def protected(plan, tw, batch, scheme="two_sided_group", delta=None, abs_floor=0.0,
              injector=None, enc=None, inverse=False, kernel="c", cap=EXEC_CAP):
    """protected.py:63-166 -> (outputs, report dict, Passes)."""
    batch = np.ascontiguousarray(batch, dtype=plan.dtype)
    if batch.ndim != 2 or batch.shape[1] != plan.n:
        raise ValueError("batch must have shape (B, n) with n == plan.n")
    total, bs = batch.shape[0], plan.bs
    if total % bs:
        raise ValueError(f"batch size {total} not divisible by group size {bs}")
    delta = default_delta(plan.precision) if delta is None else delta
    enc = enc if enc is not None else encoding_for("wang", plan.n, kernel)
    counter = Passes()
    outputs = np.empty_like(batch)
    rep = dict(scheme=scheme, delta=delta, groups=total // bs, flagged=[], corrected=[],
               unrecoverable=[], recompute_count=0, pass_count=0, max_rel_discrepancy=0.0)
    guarded = scheme != "none"
    for g, start in enumerate(range(0, total, bs)):
        xg = batch[start:start + bs]
        state = encode(xg, enc, inverse) if guarded else None
        work = xg.copy()
        hook = None
        if injector is not None:
            injector("input", start, work)

            def hook(k, view, _s=start):
                injector(f"stage:{k}", _s, view)
        yg = execute(plan, tw, work, inverse, counter, hook, kernel, cap)
        if injector is not None:
            injector("output", start, yg)
        if not guarded:
            outputs[start:start + bs] = yg
            continue
        flagged, rel, unrec = verify(state, yg, enc, delta, abs_floor, plan.precision)
        rep["max_rel_discrepancy"] = max(rep["max_rel_discrepancy"],
                                         float(np.max(rel, initial=0.0)))
        for f, r, _ in flagged:
            rep["flagged"].append({"group": g, "signal": start + f, "discrepancy": r})
        if unrec:
            rep["unrecoverable"].append(g)
        elif flagged:
            f = flagged[0][0]
            if scheme == "one_sided":
                yg = yg.copy()
                yg[f] = execute(plan, tw, xg[f], inverse, counter, None, kernel, cap)
                rep["recompute_count"] += 1
                rep["corrected"].append({"group": g, "signal": start + f})
            else:
                try:
                    yg = repair(state, yg, f, plan, tw, enc, delta, abs_floor, inverse,
                                kernel)
                    rep["corrected"].append({"group": g, "signal": start + f})
                except Unrecoverable:
                    rep["unrecoverable"].append(g)
        outputs[start:start + bs] = yg
    rep["pass_count"] = counter.total
    return outputs, rep, counter


def report_json(rep):
    """protected.py:46-60 (max_rel_discrepancy is not serialised)."""
    keys = ("scheme", "delta", "groups", "flagged", "corrected", "unrecoverable",
            "recompute_count", "pass_count")
    return json.dumps({k: rep[k] for k in keys}, sort_keys=True, separators=(",", ":"))


# --------------------------------------------------------------------------
# bit flips (fault_lab/bits.py:11-77)
# --------------------------------------------------------------------------

_UINT = {np.dtype(np.float32): np.uint32, np.dtype(np.float64): np.uint64}


def flip(value, bit):
    arr = np.asarray(value)
    if arr.dtype not in _UINT:
        arr = arr.astype(np.float64)
    width = arr.dtype.itemsize * 8
    if not 0 <= bit < width:
        raise ValueError("bit out of range")
    u = _UINT[arr.dtype]
    v = arr.copy().view(u)
    v ^= u(1) << u(bit)
    out = v.view(arr.dtype)
    return out[()] if out.ndim == 0 else out


def flip_in(buf, signal, element, component, bit):
    reals = buf.view(buf.real.dtype).reshape(buf.shape[0], -1)
    col = 2 * element + (0 if component == "re" else 1)
    reals[signal, col] = flip(reals[signal, col], bit)


class OneShot:
    """bits.py:56-77 — one-shot injector bound to a `where` point."""

    def __init__(self, signal, element, component, bit, stage="output"):
        self.signal, self.element, self.component = signal, element, component
        self.bit, self.stage, self.fired = bit, stage, False

    def __call__(self, where, start, buf):
        if self.fired or where != self.stage:
            return
        local = self.signal - start
        if not 0 <= local < buf.shape[0]:
            return
        flat = buf.reshape(buf.shape[0], -1)
        if self.element >= flat.shape[1]:
            return
        flip_in(flat, local, self.element, self.component, self.bit)
        self.fired = True
