"""Template-based kernel plan generator (paper §"code generator").

For every (precision, N) this picks the launch parameters of the sm_100a
kernels — elements per thread E (8/16/32), the radix sequence of the
in-kernel Stockham passes, CTA size and the shared-memory padding — and emits
the explicit template instantiations plus a registry the C ABI dispatches on.

The shared-memory padding is chosen by simulating the bank behaviour of every
smem exchange of the Stockham engine (csrc/engine.cuh) for each candidate
padding and keeping the cheapest. Run ``python -m paper_2405_02520_b200.codegen``
(``build()`` does it) to regenerate ``csrc/gen_*.cu``.
"""

from __future__ import annotations

import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")

# Single-kernel path (N <= 2^13): candidate launch configurations per
# (precision, log2 N) as (E, radices, threads, min CTAs/SM, staged I/O).
# Candidate 0 is the default; tools/tune.py times all of them on the B200
# and SINGLE_CHOICE records the winner (index into the candidate list).
def _cands(*rows):
    return [dict(e=r[0], radices=tuple(r[1]), threads=r[2], minb=r[3], stage=r[4]) for r in rows]


SINGLE_CANDIDATES = {
    "fp32": {
        1: _cands((2, (2,), 256, 1, 1), (2, (2,), 256, 1, 0), (2, (2,), 256, 1, 3)),
        2: _cands((4, (4,), 256, 1, 1), (4, (4,), 256, 1, 0), (4, (4,), 256, 1, 3)),
        3: _cands((8, (8,), 256, 1, 1), (8, (8,), 256, 1, 0), (4, (4, 2), 256, 1, 1),
                  (8, (8,), 128, 1, 1), (8, (8,), 128, 1, 3), (8, (8,), 256, 1, 3),
                  (4, (4, 2), 256, 1, 3)),
        4: _cands((16, (16,), 256, 1, 1), (16, (16,), 256, 1, 0), (8, (8, 2), 256, 1, 1),
                  (4, (4, 4), 256, 1, 1), (16, (16,), 128, 1, 1), (16, (16,), 128, 1, 3),
                  (8, (8, 2), 256, 1, 3)),
        5: _cands((8, (8, 4), 256, 1, 1), (8, (8, 4), 256, 1, 0), (16, (16, 2), 256, 1, 1),
                  (32, (32,), 256, 1, 1), (8, (8, 4), 256, 1, 3), (8, (8, 4), 256, 1, 2),
                  (8, (8, 4), 256, 1, 5), (8, (8, 4), 256, 2, 5), (16, (16, 2), 256, 1, 5),
                  (4, (4, 4, 2), 256, 2, 5), (8, (8, 4), 256, 3, 5),
                  # thread per signal: one in-register radix-32 DFT, no exchange / no shuffle sums
                  (32, (32,), 128, 1, 3), (32, (32,), 256, 1, 3), (32, (32,), 128, 2, 3),
                  (8, (8, 4), 256, 2, 13), (8, (8, 4), 256, 4, 5), (8, (8, 4), 256, 4, 13),
                  (32, (32,), 128, 2, 11)),
        6: _cands((8, (8, 8), 256, 1, 1), (8, (8, 8), 256, 1, 0), (16, (16, 4), 256, 1, 1),
                  (16, (16, 4), 256, 1, 0), (8, (8, 8), 256, 1, 3), (8, (8, 8), 256, 1, 2),
                  (8, (8, 8), 256, 1, 5), (8, (8, 8), 256, 2, 5), (8, (8, 8), 256, 3, 5),
                  (32, (32, 2), 128, 1, 3), (32, (32, 2), 256, 1, 3), (16, (16, 4), 256, 1, 3),
                  (16, (16, 4), 256, 2, 2),
                  # warp-shuffle transpose exchange (stage code | 16)
                  (8, (8, 8), 256, 1, 18), (8, (8, 8), 256, 3, 21)),
        7: _cands((16, (16, 8), 256, 1, 0), (16, (16, 8), 256, 1, 1), (8, (8, 8, 2), 256, 1, 0),
                  (16, (16, 8), 256, 3, 0), (16, (16, 8), 256, 1, 2), (16, (16, 8), 128, 4, 0)),
        8: _cands((16, (16, 16), 256, 1, 0), (16, (16, 16), 256, 3, 0), (8, (8, 8, 4), 256, 1, 0),
                  (16, (16, 16), 256, 1, 1), (16, (16, 16), 256, 1, 2), (16, (16, 16), 256, 3, 2),
                  (16, (16, 16), 128, 4, 0), (16, (16, 16), 128, 4, 2),
                  (16, (16, 16), 256, 1, 18), (16, (16, 16), 256, 1, 16)),
        9: _cands((16, (16, 16, 2), 256, 2, 0), (32, (32, 16), 256, 1, 0),
                  (8, (8, 8, 8), 256, 3, 0), (16, (16, 16, 2), 256, 3, 0),
                  (16, (16, 16, 2), 256, 2, 2), (8, (8, 8, 8), 256, 3, 2), (32, (32, 16), 256, 2, 0),
                  (32, (32, 16), 128, 3, 0), (16, (16, 16, 2), 128, 3, 0), (16, (16, 16, 2), 128, 4, 0)),
        10: _cands((16, (16, 16, 4), 256, 2, 0), (32, (32, 32), 256, 1, 0),
                   (16, (16, 16, 4), 256, 3, 0), (8, (8, 8, 8, 2), 256, 2, 0),
                   (16, (16, 16, 4), 512, 1, 0), (16, (16, 16, 4), 256, 3, 2),
                   (16, (16, 16, 4), 256, 2, 2), (32, (32, 32), 256, 2, 0), (32, (32, 32), 128, 2, 0),
                   (32, (32, 32), 128, 3, 0), (32, (32, 32), 128, 3, 16)),
        11: _cands((16, (16, 16, 8), 256, 2, 0), (16, (16, 16, 8), 256, 3, 0),
                   (8, (8, 8, 8, 4), 256, 3, 0), (16, (16, 16, 8), 512, 1, 0),
                   (16, (16, 16, 8), 256, 3, 2), (16, (16, 16, 8), 256, 2, 2),
                   (16, (16, 16, 8), 256, 2, 4), (32, (32, 32, 2), 128, 3, 0), (32, (32, 16, 4), 128, 3, 0),
                   (32, (32, 16, 4), 128, 2, 6), (32, (32, 32, 2), 128, 2, 6), (16, (16, 16, 8), 256, 2, 6),
                   (32, (32, 16, 4), 128, 3, 2), (32, (32, 16, 4), 128, 3, 4), (32, (32, 16, 4), 128, 2, 2),
                   (32, (32, 16, 4), 128, 2, 4),
                   (32, (16, 16, 8), 128, 3, 4), (32, (8, 16, 16), 128, 3, 4), (32, (32, 8, 8), 128, 3, 4)),
        12: _cands((16, (16, 16, 16), 256, 2, 0), (16, (16, 16, 16), 256, 3, 0),
                   (8, (8, 8, 8, 8), 512, 2, 0), (16, (16, 16, 16), 512, 1, 0),
                   (16, (16, 16, 16), 256, 3, 2), (16, (16, 16, 16), 256, 2, 2),
                   (16, (16, 16, 16), 256, 2, 4), (32, (32, 32, 4), 128, 3, 0), (32, (32, 16, 8), 128, 3, 0),
                   (16, (16, 16, 16), 256, 2, 6), (32, (32, 16, 8), 128, 2, 6),
                   (32, (32, 16, 8), 128, 3, 4), (32, (32, 16, 8), 128, 2, 4), (32, (32, 16, 8), 128, 3, 2),
                   (32, (16, 16, 16), 128, 3, 4), (32, (16, 32, 8), 128, 3, 4), (32, (8, 32, 16), 128, 3, 4),
                   (32, (32, 16, 8), 128, 3, 4 + 32), (32, (32, 16, 8), 128, 2, 4 + 32)),
        13: _cands((16, (16, 16, 16, 2), 512, 2, 0), (32, (32, 16, 16), 256, 1, 0),
                   (16, (16, 16, 16, 2), 512, 1, 0), (8, (8, 8, 8, 8, 2), 1024, 1, 0),
                   (16, (16, 16, 16, 2), 512, 2, 2), (16, (16, 16, 16, 2), 512, 1, 2),
                   (16, (16, 16, 16, 2), 512, 2, 1), (16, (16, 16, 16, 2), 512, 2, 4),
                   (16, (16, 16, 16, 2), 512, 1, 4), (16, (16, 16, 16, 2), 512, 1, 6),
                   (32, (32, 16, 16), 256, 1, 6), (32, (32, 16, 16), 256, 1, 4),
                   (32, (32, 16, 16), 256, 1, 2),
                   (32, (16, 16, 32), 256, 1, 4), (32, (16, 32, 16), 256, 1, 4), (32, (32, 32, 8), 256, 1, 4),
                   (32, (32, 16, 16), 256, 1, 4 + 32), (32, (32, 16, 16), 256, 1, 2 + 32),
                   (32, (32, 32, 8), 256, 1, 4 + 32), (16, (16, 16, 16, 2), 512, 1, 4 + 32)),
    },
    "fp64": {
        1: _cands((2, (2,), 256, 1, 1), (2, (2,), 256, 1, 0), (2, (2,), 256, 1, 3)),
        2: _cands((4, (4,), 256, 1, 1), (4, (4,), 256, 1, 0), (4, (4,), 256, 1, 3)),
        3: _cands((8, (8,), 256, 1, 1), (8, (8,), 256, 1, 0), (4, (4, 2), 256, 1, 1),
                  (8, (8,), 128, 1, 3), (8, (8,), 256, 1, 3)),
        4: _cands((16, (16,), 256, 1, 1), (8, (8, 2), 256, 1, 1), (4, (4, 4), 256, 1, 1),
                  (8, (8, 2), 256, 1, 3), (16, (16,), 128, 1, 3), (8, (8, 2), 256, 1, 5),
                  (4, (4, 4), 256, 1, 5), (8, (8, 2), 256, 2, 5)),
        5: _cands((8, (8, 4), 256, 1, 1), (8, (8, 4), 256, 1, 0), (16, (16, 2), 256, 1, 1),
                  (8, (8, 4), 256, 1, 3), (8, (8, 4), 256, 1, 2), (8, (8, 4), 256, 1, 5)),
        6: _cands((8, (8, 8), 256, 1, 1), (8, (8, 8), 256, 1, 0), (16, (16, 4), 256, 1, 0),
                  (8, (8, 8), 256, 1, 3), (8, (8, 8), 256, 1, 2)),
        7: _cands((16, (16, 8), 256, 1, 0), (8, (8, 8, 2), 256, 1, 0), (16, (16, 8), 256, 1, 1),
                  (16, (16, 8), 256, 1, 2)),
        8: _cands((16, (16, 16), 256, 1, 0), (8, (8, 8, 4), 256, 1, 0), (16, (16, 16), 256, 2, 0),
                  (16, (16, 16), 256, 2, 2), (16, (16, 16), 128, 3, 0), (16, (16, 16), 128, 4, 0)),
        9: _cands((8, (8, 8, 8), 256, 1, 0), (16, (16, 16, 2), 256, 1, 0),
                  (8, (8, 8, 8), 256, 3, 0), (8, (8, 8, 8), 256, 3, 2),
                  (8, (8, 8, 8), 256, 2, 4), (16, (16, 16, 2), 128, 2, 0), (16, (16, 16, 2), 128, 3, 0)),
        10: _cands((16, (16, 16, 4), 256, 1, 0), (8, (8, 8, 8, 2), 256, 1, 0),
                   (16, (16, 16, 4), 256, 2, 0), (16, (16, 16, 4), 256, 2, 2),
                   (16, (16, 16, 4), 256, 2, 4), (8, (8, 8, 8, 2), 256, 2, 4), (16, (16, 16, 4), 128, 3, 0),
                   (16, (16, 16, 4), 128, 2, 0)),
        11: _cands((16, (16, 16, 8), 256, 1, 0), (16, (16, 16, 8), 256, 2, 0),
                   (8, (8, 8, 8, 4), 256, 2, 0), (16, (16, 16, 8), 256, 2, 2),
                   (8, (8, 8, 8, 4), 256, 2, 4), (16, (16, 16, 8), 128, 3, 0), (16, (16, 16, 8), 128, 2, 0),
                   (16, (16, 16, 8), 256, 1, 6), (16, (16, 16, 8), 128, 1, 6),
                   (16, (16, 16, 8), 128, 2, 32), (16, (16, 16, 8), 128, 3, 32)),
        12: _cands((16, (16, 16, 16), 256, 1, 0), (16, (16, 16, 16), 512, 1, 0),
                   (8, (8, 8, 8, 8), 512, 1, 0), (16, (16, 16, 16), 256, 1, 2),
                   (16, (16, 16, 16), 256, 1, 4), (8, (8, 8, 8, 8), 512, 1, 4),
                   (8, (8, 8, 8, 8), 512, 2, 4), (16, (16, 16, 16), 256, 1, 6),
                   (16, (16, 16, 16), 256, 1, 4 + 32)),
        13: _cands((16, (16, 16, 16, 2), 512, 1, 0), (8, (8, 8, 8, 8, 2), 1024, 1, 0),
                   (16, (16, 16, 16, 2), 512, 1, 4), (8, (8, 8, 8, 8, 2), 1024, 1, 4)),
    },
}
# tuned winners (index into SINGLE_CANDIDATES[prec][logn]); missing -> 0.
# Source: tools/tune.py on a B200, ABFT on, 1 GiB batches (profiles/tune_r01.json).
# Round 2 (profiles/tune_r02_fp32.json, tune_r02_fp64.json; timed at a delta with no
# clean-data false alarms): fp32 N = 32 -> 2 CTAs/SM, N = 1024 -> 3 CTAs/SM,
# N = 8192 -> E = 32 in 256-thread CTAs (in-place TMA prefetch); fp64: the
# full retune after the addressing rewrite left every choice within 1-2 %
# (profiles/tune_r02h_fp64.json; N = 2048 back to 3 CTAs/SM, direct loads); after the exchange-addressing
# rewrite (profiles/tune_r02c_fp32.json) N = 64 -> TMA bulk prefetch (STAGE 2);
# N = 32 -> e^T W row read from smem each tile (stage code 13: 0.420 -> 0.407
# ms, profiles/tune_r02e_fp32.json; the thread-per-signal radix-32 variants
# measured 0.436); N = 2048 / 4096 -> E = 32 in 128-thread CTAs, 3 per SM, with
# the in-place TMA prefetch (0.473 -> 0.423 / 0.444 -> 0.424 ms,
# profiles/tune_r02f_fp32.json).
SINGLE_CHOICE = {
    "fp32": {1: 1, 2: 1, 3: 4, 4: 5, 5: 17, 6: 8, 7: 0, 8: 4, 9: 7, 10: 9, 11: 18, 12: 13, 13: 16},
    "fp64": {1: 1, 2: 2, 3: 3, 4: 7, 5: 5, 6: 4, 7: 0, 8: 4, 9: 6, 10: 4, 11: 7, 12: 8, 13: 2},
}
# One-loop twins (stage code | 64, single.cuh ONE_LOOP) of the tuned configs:
# the single kernel instantiates its tile loop per direction and once more for
# fault injection; these sizes measured faster with ONE runtime loop (fewer
# registers, more CTAs per SM) — A/B in profiles/ab_loop_r02.json.
ONE_LOOP_SIZES = {"fp32": (4, 7, 8), "fp64": (1, 5, 6, 13)}
for _p, _sizes in ONE_LOOP_SIZES.items():
    for _l in _sizes:
        _twin = dict(SINGLE_CANDIDATES[_p][_l][SINGLE_CHOICE[_p][_l]])
        _twin["stage"] |= 64
        SINGLE_CANDIDATES[_p][_l].append(_twin)
        SINGLE_CHOICE[_p][_l] = len(SINGLE_CANDIDATES[_p][_l]) - 1
ELEM_BYTES = {"fp32": 8, "fp64": 16}
CTYPE = {"fp32": "float", "fp64": "double"}


def _pad(i, ps):
    return i if ps == 0 else i + (i >> ps)


def _wavefronts(addrs, elem_bytes):
    """Shared-memory wavefronts for one warp access of `elem_bytes` elements.

    A warp request is split into phases of 128 bytes (16 lanes for 8-byte,
    8 lanes for 16-byte elements); within a phase, the cost is the largest
    number of distinct 4-byte words that fall into one of the 32 banks.
    """
    lanes_per_phase = 128 // elem_bytes
    words = elem_bytes // 4
    total = 0
    for p in range(0, 32, lanes_per_phase):
        banks = {}
        for a in addrs[p:p + lanes_per_phase]:
            if a is None:
                continue
            for w in range(words):
                word = a * words + w
                banks.setdefault(word % 32, set()).add(word)
        total += max((len(s) for s in banks.values()), default=0)
    return total


def smem_cost(n, e, radices, ps, elem_bytes):
    """Total wavefronts of all smem exchanges of one CTA's first warps."""
    tps = n // e
    slen = n + (n >> ps) + 1 if ps else n
    warps = max(1, tps // 32)
    cost = 0
    ns = 1
    for r in radices[:-1]:
        sub = e // r
        for w in range(warps):
            lanes = [divmod(32 * w + lane, tps) for lane in range(32)]
            for q in range(sub):
                for rr in range(r):
                    addrs = []
                    for sig, tt in lanes:
                        j = tt + q * tps
                        o = (j // ns) * ns * r + (j % ns) + rr * ns
                        addrs.append(sig * slen + _pad(o, ps))
                    cost += _wavefronts(addrs, elem_bytes)
            for m in range(e):
                addrs = [sig * slen + _pad(tt + m * tps, ps) for sig, tt in lanes]
                cost += _wavefronts(addrs, elem_bytes)
        ns *= r
    return cost


def choose_padding(n, e, radices, prec):
    if len(radices) == 1:
        return 0, 0
    best = None
    for ps in (0, 5, 4, 3, 2):
        c = smem_cost(n, e, radices, ps, ELEM_BYTES[prec])
        if best is None or c < best[1]:
            best = (ps, c)
    return best


def tune_sizes():
    """TFFT_TUNE_SIZES="fp32:11,12,13;fp64:12" limits the tuning build's extra
    candidates to those sizes (every other size keeps its chosen kernel)."""
    spec = os.environ.get("TFFT_TUNE_SIZES", "")
    if not spec:
        return None
    out = set()
    for part in spec.split(";"):
        prec, sizes = part.split(":")
        out.update((prec, int(v)) for v in sizes.split(","))
    return out


def single_configs(all_candidates=True):
    """Every candidate (all_candidates) or only the chosen one per size."""
    out = []
    only = tune_sizes() if all_candidates else None
    for prec, table in SINGLE_CANDIDATES.items():
        for logn, cands in sorted(table.items()):
            chosen = SINGLE_CHOICE[prec].get(logn, 0)
            for vi, c in enumerate(cands):
                if (not all_candidates or (only is not None and (prec, logn) not in only)) and vi != chosen:
                    continue
                n = 1 << logn
                e, radices = c["e"], c["radices"]
                assert math.prod(radices) == n and all(e % r == 0 for r in radices), (prec, logn, c)
                tps = n // e
                threads = max(c["threads"], tps)
                ps, _ = choose_padding(n, e, radices, prec)
                s = threads // tps
                ex = (n + (n >> ps) + 1 if ps else n) if len(radices) > 1 else 0
                ld = c["stage"] & 7  # load strategy (| 8 / | 32: e^T W row from static / dynamic smem)
                st = n + 1 if ld in (1, 3) else (n if ld == 4 else 0)
                ib = s * n if ld in (2, 3, 6) else 0  # TMA prefetch buffer
                if ld == 5:  # per-signal rows into padded slots
                    ib = s * (n + 32 // ELEM_BYTES[prec])
                # ABFT scratch: per-warp sums (TPS <= 32) or the deferred
                # two-tile reduction pipeline (2 x S x 5 x TPS partials + totals)
                # (sized for >= 64-thread signals: TFFT_DEFER_MIN may select the pipeline there)
                red = 10 * (threads // 32 + 1) + (10 * threads + 10 * s if tps >= 64 else 0)
                regions = 2 if ld == 6 else 1  # ping-pong exchange regions
                smem = (ib + regions * s * max(ex, st)) * ELEM_BYTES[prec] + red * (ELEM_BYTES[prec] // 2)
                if c["stage"] & 32:  # e^T W row behind the (16-byte rounded) ABFT scratch
                    smem += ((red + 3) // 4 * 4 - red) * (ELEM_BYTES[prec] // 2) + n * ELEM_BYTES[prec]
                out.append(dict(prec=prec, logn=logn, n=n, e=e, radices=radices, threads=threads,
                                ps=ps, smem=smem, tps=tps, minb=c["minb"], stage=c["stage"],
                                variant=vi, chosen=vi == chosen))
    return out


def _emit_single(prec, cfgs, part, table=False):
    t = CTYPE[prec]
    lines = [
        "// GENERATED by paper_2405_02520_b200/codegen.py — do not edit.",
        '#include "fix.cuh"',
        '#include "registry.h"',
        "namespace tfft {",
    ]
    entries = []
    for c in cfgs:
        rl = ", ".join(str(r) for r in c["radices"])
        fns = []
        for abft in (0, 1, 2, 3):
            if abft >= 2 and not c["chosen"]:
                fns.append("nullptr")  # table / thread-level checks only on the chosen config
                continue
            fns.append(f"(const void*)&fft_single_kernel<{t}, {c['n']}, {c['e']}, {c['ps']}, "
                       f"{abft}, {c['threads']}, {c['minb']}, {c['stage']}, RList<{rl}>>")
        fix = "nullptr, 0, 0"
        if c["chosen"]:  # device-side correction with the same engine config (fix.cuh)
            ft = max(c["tps"], 32)
            fsl = (c["n"] + (c["n"] >> c["ps"]) + 1 if c["ps"] else c["n"]) if len(c["radices"]) > 1 else 1
            fix = (f"(const void*)&fix_single_kernel<{t}, {c['n']}, {c['e']}, {c['ps']}, {ft}, RList<{rl}>>, "
                   f"{ft}, {(ft // c['tps']) * fsl * ELEM_BYTES[prec]}")
        entries.append(
            f"    {{{c['logn']}, {c['variant']}, {int(c['chosen'])}, {c['e']}, {c['threads']}, "
            f"{c['smem']}, {c['tps']}, {c['stage']}, {{{', '.join(fns)}}}, {fix}}},  // radices {rl}, "
            f"pad 2^{c['ps']}, minb {c['minb']}, stage {c['stage']}")
    lines.append(f"extern const SingleEntry kSingle_{prec}_{part}[] = {{")
    lines += entries
    lines.append("};")
    lines.append(f"extern const int kSingleCount_{prec}_{part} = {len(cfgs)};")
    lines.append("}  // namespace tfft")
    return "\n".join(lines) + "\n"


SINGLE_PARTS = 4


def _emit_single_index(parts):
    lines = ["// GENERATED by paper_2405_02520_b200/codegen.py — do not edit.",
             '#include "registry.h"', "namespace tfft {"]
    for prec in ("fp32", "fp64"):
        for p in range(parts):
            lines.append(f"extern const SingleEntry kSingle_{prec}_{p}[];")
            lines.append(f"extern const int kSingleCount_{prec}_{p};")
        lines.append(f"const SingleTable kSingleTables_{prec}[] = {{"
                     + ", ".join(f"{{kSingle_{prec}_{p}, &kSingleCount_{prec}_{p}}}"
                                 for p in range(parts)) + "};")
    lines.append(f"const int kSingleParts = {parts};")
    lines.append("}  // namespace tfft")
    return "\n".join(lines) + "\n"


# Multi-pass tile kernels (one launch per reference stage): candidates per
# (precision, log2 L) as (E, radices, U, min CTAs/SM, prefetch), U = tile
# width in transforms (row segment = U * sizeof(complex) bytes). Small L only
# occur in user-built plans and keep one config. PASS_CHOICE picks a variant
# per stage kind (first, middle, last) from tools/tune_pass.py.
def _pc(*rows):
    return [dict(e=r[0], radices=tuple(r[1]), u=r[2], minb=r[3], pf=r[4]) for r in rows]


PASS_CANDIDATES = {
    "fp32": {
        1: _pc((2, (2,), 16, 1, 0)), 2: _pc((4, (4,), 16, 1, 0)), 3: _pc((8, (8,), 16, 1, 0)),
        4: _pc((16, (16,), 16, 1, 0)), 5: _pc((8, (8, 4), 16, 1, 0)),
        6: _pc((8, (8, 8), 16, 1, 0), (8, (8, 8), 32, 2, 3), (8, (8, 8), 16, 3, 3), (8, (8, 8), 32, 2, 2),
               (8, (8, 8), 16, 3, 2), (8, (8, 8), 32, 2, 4), (8, (8, 8), 16, 3, 4)),
        7: _pc((16, (16, 8), 16, 1, 0), (16, (16, 8), 16, 2, 1), (16, (16, 8), 8, 3, 1),
               (8, (8, 8, 2), 16, 2, 1), (16, (16, 8), 16, 2, 2), (16, (16, 8), 8, 3, 2),
               (16, (16, 8), 16, 2, 3), (16, (16, 8), 8, 3, 3), (16, (16, 8), 32, 1, 3),
               (16, (16, 8), 16, 2, 4), (16, (16, 8), 8, 3, 4),
               (32, (32, 4), 16, 3, 3), (32, (32, 4), 32, 2, 3), (32, (32, 4), 16, 3, 2),
               (32, (32, 4), 32, 2, 4)),
        8: _pc((16, (16, 16), 16, 1, 0), (16, (16, 16), 16, 2, 1), (16, (16, 16), 8, 3, 1),
               (16, (16, 16), 8, 2, 0), (16, (16, 16), 16, 2, 2), (16, (16, 16), 8, 3, 2),
               (16, (16, 16), 16, 2, 3), (16, (16, 16), 8, 3, 3), (16, (16, 16), 16, 2, 4),
               (32, (32, 8), 16, 2, 3), (32, (32, 8), 8, 3, 3), (32, (32, 8), 16, 2, 2)),
        9: _pc((16, (16, 16, 2), 16, 1, 0), (16, (16, 16, 2), 8, 2, 1), (16, (16, 16, 2), 4, 3, 1),
               (16, (16, 16, 2), 8, 2, 0), (16, (16, 16, 2), 8, 2, 2), (16, (16, 16, 2), 16, 1, 2),
               (16, (16, 16, 2), 16, 1, 3), (16, (16, 16, 2), 8, 2, 3),
               (32, (32, 16), 8, 2, 3), (32, (32, 16), 16, 1, 3), (32, (32, 16), 8, 2, 2),
               (32, (32, 16), 4, 3, 2)),
        10: _pc((16, (16, 16, 4), 8, 1, 0), (16, (16, 16, 4), 4, 2, 1), (16, (16, 16, 4), 4, 3, 0),
                (32, (32, 32), 8, 1, 1), (16, (16, 16, 4), 8, 1, 1), (16, (16, 16, 4), 8, 1, 2),
                (16, (16, 16, 4), 4, 2, 2), (16, (16, 16, 4), 8, 1, 3), (16, (16, 16, 4), 4, 2, 3),
                (32, (32, 32), 8, 1, 3), (32, (32, 32), 4, 2, 2), (32, (32, 32), 4, 2, 3),
                (32, (32, 32), 8, 1, 2)),
        11: _pc((16, (16, 16, 8), 4, 1, 0), (16, (16, 16, 8), 4, 2, 1), (16, (16, 16, 8), 2, 3, 1),
                (32, (32, 16, 4), 4, 1, 1), (16, (16, 16, 8), 4, 1, 2), (16, (16, 16, 8), 2, 2, 2),
                (16, (16, 16, 8), 4, 1, 3), (16, (16, 16, 8), 2, 2, 3)),
    },
    "fp64": {
        1: _pc((2, (2,), 8, 1, 0)), 2: _pc((4, (4,), 8, 1, 0)), 3: _pc((8, (8,), 8, 1, 0)),
        4: _pc((16, (16,), 8, 1, 0)), 5: _pc((8, (8, 4), 8, 1, 0)),
        6: _pc((8, (8, 8), 8, 1, 0), (8, (8, 8), 16, 2, 3), (8, (8, 8), 8, 3, 3), (8, (8, 8), 16, 2, 2),
               (8, (8, 8), 8, 3, 2), (8, (8, 8), 16, 2, 4),
               (16, (16, 4), 16, 2, 3), (16, (16, 4), 8, 3, 3), (16, (16, 4), 16, 2, 4)),
        7: _pc((16, (16, 8), 8, 1, 0), (16, (16, 8), 8, 2, 1), (16, (16, 8), 4, 3, 1),
               (8, (8, 8, 2), 8, 2, 1), (16, (16, 8), 8, 2, 2), (16, (16, 8), 4, 3, 2),
               (16, (16, 8), 8, 2, 3), (16, (16, 8), 4, 3, 3), (16, (16, 8), 16, 1, 3),
               (16, (16, 8), 16, 1, 4), (16, (16, 8), 8, 2, 4),
               (32, (32, 4), 8, 2, 3), (32, (32, 4), 16, 1, 3), (32, (32, 4), 8, 2, 2)),
        8: _pc((16, (16, 16), 8, 1, 0), (16, (16, 16), 8, 2, 1), (16, (16, 16), 4, 2, 1),
               (8, (8, 8, 4), 8, 2, 1), (16, (16, 16), 8, 2, 2), (8, (8, 8, 4), 8, 2, 2),
               (16, (16, 16), 8, 2, 3), (8, (8, 8, 4), 8, 2, 3), (16, (16, 16), 8, 2, 4),
               (32, (32, 8), 8, 1, 3), (32, (32, 8), 4, 2, 3), (32, (32, 8), 8, 1, 2),
               (32, (32, 8), 4, 2, 2)),
        9: _pc((8, (8, 8, 8), 8, 1, 0), (8, (8, 8, 8), 4, 2, 1), (16, (16, 16, 2), 4, 2, 1),
               (8, (8, 8, 8), 8, 1, 1), (8, (8, 8, 8), 8, 1, 2), (8, (8, 8, 8), 4, 2, 2),
               (8, (8, 8, 8), 8, 1, 3), (8, (8, 8, 8), 4, 2, 3),
               (16, (16, 16, 2), 4, 2, 2), (16, (16, 16, 2), 8, 1, 2), (32, (32, 16), 4, 2, 2),
               (32, (32, 16), 8, 1, 2), (32, (32, 16), 4, 3, 2)),
        10: _pc((8, (8, 8, 8, 2), 8, 1, 0), (8, (8, 8, 8, 2), 4, 2, 1), (16, (16, 16, 4), 4, 1, 1),
                (16, (16, 16, 4), 2, 2, 1), (8, (8, 8, 8, 2), 4, 1, 2), (8, (8, 8, 8, 2), 2, 2, 2),
                (8, (8, 8, 8, 2), 4, 1, 3), (8, (8, 8, 8, 2), 2, 2, 3)),
        11: _pc((8, (8, 8, 8, 4), 4, 1, 0), (8, (8, 8, 8, 4), 2, 2, 1), (16, (16, 16, 8), 2, 1, 1),
                (16, (16, 16, 8), 4, 1, 0), (8, (8, 8, 8, 4), 2, 1, 2), (8, (8, 8, 8, 4), 2, 2, 2),
                (8, (8, 8, 8, 4), 2, 1, 3), (8, (8, 8, 8, 4), 2, 2, 3)),
    },
}
# (first, middle, last) variant per log2 L; missing -> (0, 0, 0).
# Source: tools/tune_pass.py on a B200, ABFT on, 1 GiB (profiles/tune_pass_r01.json);
# round 2: fp64 L = 512 last pass -> E = 16 (16, 16, 2), U = 4, bulk rows
# (fp64 2^25 transform 1.462 -> 1.377 ms per GiB, profiles/tune_pass_fp64_25.json);
# fp32 L = 256 / 512 / 1024 -> E = 32 tiles (fp32 2^17 1.135 -> 0.961 ms, 2^19
# 1.206 -> 1.094 ms per GiB, profiles/tune_pass_fp32_16.json); fp32 L = 128
# middle / last -> E = 32 (2^21 -3 %, 2^14 -3 %, profiles/tune_pass_fp32_14.json,
# tune_pass_fp32_21.json), L = 256 middle -> TMA prefetch PF 4 (2^24 -1.5 %);
# fp64 L = 256 last -> E = 32 (2^16 -2.9 %, 2^22 -1.0 %, tune_pass_fp64_16b.json /
# tune_pass_fp64_20.json: every other fp64 choice stayed the best).
PASS_CHOICE = {
    "fp32": {6: (6, 2, 4), 7: (9, 12, 11), 8: (9, 9, 10), 9: (9, 0, 10), 10: (7, 0, 9), 11: (6, 0, 6)},
    "fp64": {6: (5, 5, 0), 7: (8, 8, 8), 8: (6, 6, 11), 9: (2, 0, 8), 10: (6, 0, 6), 11: (0, 0, 3)},
}


def tile_cost(l, e, radices, u, p, elem_bytes):
    """Wavefronts of the multi-pass tile's smem traffic (engine + staging)."""
    tps = l // e
    rs = u + p
    threads = u * tps
    cost = 0
    ns = 1
    for w in range(min(threads // 32, 8) or 1):
        lanes = [((32 * w + lane) % u, (32 * w + lane) // u) for lane in range(32)]
        ns = 1
        for r in radices[:-1]:
            sub = e // r
            for q in range(sub):
                for rr in range(r):
                    addrs = []
                    for uu, t in lanes:
                        j = t + q * tps
                        o = (j // ns) * ns * r + (j % ns) + rr * ns
                        addrs.append(o * rs + uu)
                    cost += _wavefronts(addrs, elem_bytes)
            for m in range(e):
                cost += _wavefronts([(t + m * tps) * rs + uu for uu, t in lanes], elem_bytes)
            ns *= r
        # last-kind staging store (j fastest) and gather (u fastest)
        for f0 in range(32 * w, u * l, threads):
            addrs = [((f0 + lane) % l) * rs + (f0 + lane) // l for lane in range(32)]
            cost += _wavefronts(addrs, elem_bytes)
        for m in range(e):
            cost += _wavefronts([(t + m * tps) * rs + uu for uu, t in lanes], elem_bytes)
    return cost


def pass_configs(all_candidates=True):
    """Every candidate (all_candidates) or only variant 0 (the fallback) and
    the tuned (first, middle, last) choices per stage dim."""
    out = []
    for prec, table in PASS_CANDIDATES.items():
        eb = ELEM_BYTES[prec]
        for logl, cands in sorted(table.items()):
            keep = {0, *PASS_CHOICE[prec].get(logl, (0, 0, 0))}
            for vi, c in enumerate(cands):
                if not all_candidates and vi not in keep:
                    continue
                l = 1 << logl
                e, radices = c["e"], c["radices"]
                assert math.prod(radices) == l and all(e % r == 0 for r in radices), (prec, logl, c)
                tps = l // e
                u = max(c["u"], 32 // tps)  # whole warps: the tile reductions use full-warp shuffles
                threads = u * tps
                assert threads <= 1024, (prec, logl, c)
                best = min((tile_cost(l, e, radices, u, p, eb), p) for p in (1, 0, 2, 3, 4, 5, 8))
                p = best[1]
                nbuf = 2 if c["pf"] else 1
                bufe = l * (u + p)
                if c["pf"] in (2, 3, 4):  # bulk staging: last-kind rows at a padded stride
                    su = l + 2 if prec == "fp32" else l + 1
                    bufe = max(bufe, u * su)
                bufe = (bufe + 15) // 16 * 16  # keeps the second buffer 128-byte aligned
                etwe = (l * u + 15) // 16 * 16 if c["pf"] == 4 else 0  # e^T W tiles (first pass)
                smem = nbuf * bufe * eb + 2 * etwe * eb + 3 * (threads // 32 + 1) * (eb // 2)
                out.append(dict(prec=prec, logl=logl, l=l, e=e, radices=radices, u=u, p=p,
                                threads=threads, smem=smem, minb=c["minb"], pf=c["pf"], variant=vi))
    return out


def _emit_pass(prec, cfgs):
    t = CTYPE[prec]
    lines = [
        "// GENERATED by paper_2405_02520_b200/codegen.py — do not edit.",
        '#include "multi.cuh"',
        "namespace tfft {",
    ]
    entries = []
    for c in cfgs:
        rl = ", ".join(str(r) for r in c["radices"])

        def fn(kind, abft):
            return (f"(const void*)&fft_pass_kernel<{t}, {c['l']}, {c['e']}, {c['u']}, {c['p']}, "
                    f"{kind}, {abft}, {c['minb']}, {c['pf']}, RList<{rl}>>")
        rows = [
            f"{{{fn(0, 0)}, {fn(0, 1)}, {fn(0, 2)}}}",  # Wang: closed-form row; table encodings read it
            f"{{{fn(1, 0)}, nullptr, nullptr}}",
            f"{{{fn(2, 0)}, {fn(2, 1)}, {fn(2, 2)}}}",
        ]
        entries.append(
            f"    {{{c['logl']}, {c['variant']}, {c['pf']}, {c['e']}, {c['u']}, {c['p']}, {c['threads']}, "
            f"{c['smem']}, {{{', '.join(rows)}}}}},  // radices {rl}, minb {c['minb']}, pf {c['pf']}")
    lines.append(f"const PassEntry kPass_{prec}[] = {{")
    lines += entries
    lines.append("};")
    lines.append(f"const int kPassCount_{prec} = {len(cfgs)};")
    choice = PASS_CHOICE[prec]
    lines.append(f"const int kPassChoice_{prec}[12][3] = {{")
    for logl in range(12):
        ch = choice.get(logl, (0, 0, 0))
        lines.append(f"    {{{ch[0]}, {ch[1]}, {ch[2]}}},")
    lines.append("};")
    lines.append("}  // namespace tfft")
    return "\n".join(lines) + "\n"


def _write(path, text):
    old = open(path).read() if os.path.exists(path) else None
    if old != text:
        with open(path, "w") as f:
            f.write(text)


def wang_etw_header():
    """Constants of the thread-level check (ABFT_THREAD): e^T W of the Wang
    weights e_k = w3^(k mod 3) for one radix-R tile, etw_R[r] = sum_k e_k
    w_R^(r k), rounded once from 50-digit arithmetic."""
    try:
        import mpmath as mp
        mp.mp.dps = 50

        def etw(R, r):
            z = sum(mp.expjpi(-mp.mpf(2) * (k % 3) / 3) * mp.expjpi(-mp.mpf(2) * r * k / R) for k in range(R))
            return float(mp.re(z)), float(mp.im(z))
    except ImportError:  # pragma: no cover - long double fallback
        import numpy as np

        def etw(R, r):
            k = np.arange(R, dtype=np.longdouble)
            ang = -2 * np.pi * ((k % 3) / 3 + r * k / R)
            return float(np.cos(ang).sum()), float(np.sin(ang).sum())
    lines = ["// GENERATED by paper_2405_02520_b200/codegen.py (wang_etw_header) — do not edit.",
             "// Thread-level ABFT: e^T W of the Wang weights for one radix-R tile,",
             "// etw_R[r] = sum_k w3^(k mod 3) w_R^(r k), rounded once from 50 digits.",
             "// Constexpr lookups: with unrolled (compile-time) r they fold to immediates.",
             "#pragma once", "namespace tfft {"]
    for part, name in ((0, "re"), (1, "im")):
        lines.append(f"__host__ __device__ constexpr double wang_etw_{name}(int R, int r) {{")
        for R in (2, 4, 8, 16, 32):
            vals = [etw(R, r)[part] for r in range(R)]
            lines.append(f"    constexpr double t{R}[{R}] = {{{', '.join(repr(v) for v in vals)}}};")
        lines.append("    return R == 2 ? t2[r] : R == 4 ? t4[r] : R == 8 ? t8[r] : R == 16 ? t16[r] : t32[r];")
        lines.append("}")
    # cot(m pi / E) for the closed-form e^T W of the multi-pass first pass
    # (consecutive elements of a thread are pi/E apart in angle, multi.cuh)
    try:
        import mpmath as mp
        mp.mp.dps = 50
        cot = lambda m, e: float(mp.cot(mp.pi * m / e))  # noqa: E731
    except ImportError:  # pragma: no cover
        import numpy as np
        cot = lambda m, e: float(1 / np.tan(np.longdouble(np.pi) * m / e))  # noqa: E731
    lines.append("// cot(m pi / E), m = 1..E-1 (index 0 unused), rounded once from 50 digits.")
    lines.append("__host__ __device__ constexpr double cot_pi_frac(int E, int m) {")
    for e in (2, 4, 8, 16, 32):
        vals = [0.0] + [cot(m, e) for m in range(1, e)]
        lines.append(f"    constexpr double c{e}[{e}] = {{{', '.join(repr(v) for v in vals)}}};")
    lines.append("    return E == 2 ? c2[m] : E == 4 ? c4[m] : E == 8 ? c8[m] : E == 16 ? c16[m] : c32[m];")
    lines.append("}")
    lines.append("}  // namespace tfft")
    return "\n".join(lines) + "\n"


def tuning_build() -> bool:
    """TFFT_TUNE=1 compiles every tuning candidate (tools/tune*.py); the
    product build carries only the tuned kernels (+ pass variant 0, the
    fallback)."""
    return os.environ.get("TFFT_TUNE", "0") == "1"


def generate(verbose=False, all_candidates=None):
    if all_candidates is None:
        all_candidates = tuning_build()
    cfgs = single_configs(all_candidates)
    written = []
    path = os.path.join(CSRC, "wang_etw.cuh")
    _write(path, wang_etw_header())
    written.append(path)
    for old in ("gen_single_fp32.cu", "gen_single_fp64.cu"):
        if os.path.exists(os.path.join(CSRC, old)):
            os.remove(os.path.join(CSRC, old))
    path = os.path.join(CSRC, "gen_single_index.cu")
    _write(path, _emit_single_index(SINGLE_PARTS))
    written.append(path)
    for prec in ("fp32", "fp64"):
        mine = [c for c in cfgs if c["prec"] == prec]
        # round-robin by size so the parts compile in similar time
        for p in range(SINGLE_PARTS):
            part = [c for i, c in enumerate(mine) if c["logn"] % SINGLE_PARTS == p]
            path = os.path.join(CSRC, f"gen_single_{prec}_{p}.cu")
            _write(path, _emit_single(prec, part, p))
            written.append(path)
        pcfgs = [c for c in pass_configs(all_candidates) if c["prec"] == prec]
        path = os.path.join(CSRC, f"gen_pass_{prec}.cu")
        _write(path, _emit_pass(prec, pcfgs))
        written.append(path)
    if verbose:
        for c in cfgs:
            print(c)
    return written


if __name__ == "__main__":
    generate(verbose=True)
